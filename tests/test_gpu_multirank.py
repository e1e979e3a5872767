"""Multi-GPU parity (NCCL over NVLink): torchrun ranks vs the oracle's R-rank
emulation.  Needs >= 2 visible GPUs (run through `gpurun --gpus 2|4`); skipped
otherwise.  The host-side protocol is also covered on CPU by
tests/test_multirank_gloo.py."""
import os
import subprocess
import sys

import pytest

from tests.conftest import gpu_available

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ngpu():
    if not gpu_available():
        return 0
    import torch
    return torch.cuda.device_count()


@pytest.mark.parametrize("K,bcz,observe", [(1, 1, "each"), (2, 1, "each"), (1, 0, "each"), (2, 1, "end"),
                                           (1, 0, "end")])
def test_multigpu_matches_emulation(K, bcz, observe):
    """observe = "each": migration counts read after every call (each due rebin is flushed
    by that observation, standalone); "end": nothing observed in between, so every rebin
    runs fused into the next call's k_fs launch (multi-rank send buffers, arrivals)."""
    n = _ngpu()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    world = min(n, 4)
    env = dict(os.environ, MR_K=str(K), MR_BCZ=str(bcz), MR_STEPS=str(6 if observe == "each" else 7),
               MR_OBSERVE=observe)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(29500 + 7 * K + bcz + (50 if observe == "end" else 0)),
           os.path.join(ROOT, "tests", "mr_worker.py")]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    assert "MR_REPORT" in out


def test_multigpu_far_tails_and_arrivals_in_boundary_bins():
    """K = 4 in a flow fast along x and slow along z: far particles (C-15b) land in every
    plane, the slab's boundary planes included, in the same rebin as arrivals from the
    neighbour ranks.  Each boundary bin must come out as local runs | arrivals | far tail
    (the oracle's (bin, far) sort of kept ++ arrivals), with no slot written twice."""
    n = _ngpu()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    world = min(n, 4)
    env = dict(os.environ, MR_K="4", MR_BCZ="1", MR_STEPS="9", MR_FIELD="xshear", MR_OBSERVE="end")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", "29770", os.path.join(ROOT, "tests", "mr_worker.py")]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    assert "MR_REPORT" in out


def test_sharded_rebalance_equalises_counts():
    """f4: st_rebalance moves the surplus of the heavier ranks (15000 + 2000 r
    injected) so every rank ends with total/G particles; the physics is unchanged (the
    same single-oracle comparison as without rebalancing) and no particle is lost."""
    n = _ngpu()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    world = min(n, 4)
    env = dict(os.environ, MR_K="2", MR_STEPS="6", MR_REBALANCE="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", "29780", os.path.join(ROOT, "tests", "mr_shard_worker.py")]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    assert "MR_REPORT" in out


def test_multigpu_far_particles_across_ranks_stay_fused():
    """K = 4, fast along x everywhere and upwards: far particles (C-15b) also change rank.
    They are counted per cell of the neighbour's window by the in-place step, sent after
    the near movers, sorted by the sender's store order and put in the receiver's far
    tails — the rebin stays fused (no general sort) and the order equals the oracle's
    (bin, far) sort of kept ++ arrivals."""
    n = _ngpu()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    world = min(n, 4)
    env = dict(os.environ, MR_K="4", MR_BCZ="1", MR_STEPS="9", MR_FIELD="xcross", MR_OBSERVE="end")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", "29790", os.path.join(ROOT, "tests", "mr_worker.py")]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    assert "MR_REPORT" in out


@pytest.mark.parametrize("K,equal", [(1, False), (2, False), (2, True)])
def test_sharded_decomposition_matches_one_oracle(K, equal):
    """ST_DECOMP_SHARDED: whole domain per rank, particles stay where
    injected, sources all-reduced — equal to one oracle run holding all particles."""
    n = _ngpu()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    world = min(n, 4)
    env = dict(os.environ, MR_K=str(K), MR_STEPS="6", MR_DZ=str(16 * world if equal else 40))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(29700 + K + (10 if equal else 0)),
           os.path.join(ROOT, "tests", "mr_shard_worker.py")]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    assert "MR_REPORT" in out


def test_multigpu_weighted_slabs_match_emulation():
    """Count-balanced slab boundaries (st_plan_partition, f4): unequal slabs through the
    fused rebin, migration and halos match the oracle's emulation with the same split."""
    n = _ngpu()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    world = min(n, 4)
    env = dict(os.environ, MR_K="2", MR_BCZ="1", MR_STEPS="6", MR_SPLIT="weighted")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", "29750", os.path.join(ROOT, "tests", "mr_worker.py")]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    assert "MR_REPORT" in out


def test_collective_failure_is_collective():
    """A collective call failing on one rank raises on every rank (no hang)."""
    n = _ngpu()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", "29760", os.path.join(ROOT, "tests", "mr_error_worker.py")]
    r = subprocess.run(cmd, env=dict(os.environ), capture_output=True, text=True, timeout=300)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    assert out.count("ok=True") == 2, out[-2000:]
