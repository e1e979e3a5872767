"""torchrun worker: a collective call that fails on one rank fails on every rank (no
hang): rank 1 injects a particle outside its slab; every rank must get an StError from
st_inject, nothing is appended anywhere, and the job continues (advance + sources)."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import synth
    from paper_2603_26691_b200 import Config, ScaleTrack, StError, nccl_unique_id

    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
    uid = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    dims, h = (32, 24, 32 * world), 1 / 16
    st = ScaleTrack(Config(dims=dims, cell_size=(h, h, h), chunk_cells=8, bc=(1, 1, 1), capacity=50_000,
                           device=rank, rank=rank, nranks=world), unique_id=uid[0])
    lay = st.layout
    L = [d * h for d in dims]
    x, u, d, w = synth.particles_np(1000, (0, 0, lay.z0 * h), (L[0], L[1], lay.z1 * h), (5e-6, 40e-6), seed=5 + rank)
    st.inject(x, u, d, w)
    bad = x.copy()
    if rank == 1:
        bad[2, 0] = ((lay.z0 - 1) % dims[2]) * h + 0.5 * h   # a cell of another rank
    failed = False
    try:
        st.inject(bad, u, d, w)
    except StError:
        failed = True
    ok = failed and st.count() == 1000
    F = np.zeros((3, lay.z1 - lay.z0, dims[1], dims[0]), np.float32)
    st.set_fluid_field(F)
    for _ in range(3):
        st.advance(1e-3, 1)
    S, T = st.get_sources()
    ok &= st.count() == 1000 and T > 0
    print(f"MR_ERR rank {rank} failed={failed} n={st.count()} ok={ok}", flush=True)
    st.close()
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(0 if ok else 3)


if __name__ == "__main__":
    main()
