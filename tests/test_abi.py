"""CPU-side checks of the C-ABI boundary: the library loads, exports every symbol
include/scaletrack.h declares, its ctypes mirrors match the C struct sizes, and
(without a GPU) st_init fails loudly instead of falling back to the CPU."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "scaletrack.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(st_[a-z_0-9]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_2603_26691_b200 import _native
    return _native.load()


def test_every_declared_symbol_is_exported(lib):
    from paper_2603_26691_b200 import _native
    names = declared_functions()
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), n
        assert n in _native.SIGNATURES, f"binding misses {n}"
    out = subprocess.run(["nm", "-D", "--defined-only", _native.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (st_[a-z_0-9]+)", out))
    assert set(names) <= exported


def test_struct_layouts_match_header():
    """sizeof/offsetof of st_config, st_layout, st_stats computed by the C compiler."""
    from paper_2603_26691_b200 import _native as N
    prog = r'''
#include <stdio.h>
#include <stddef.h>
#include "scaletrack.h"
int main(void){
  printf("%zu %zu %zu %zu %zu %zu %zu\n", sizeof(st_config), sizeof(st_layout), sizeof(st_stats),
         offsetof(st_config, capacity), offsetof(st_config, stream), offsetof(st_config, nccl_unique_id),
         offsetof(st_layout, local_cells));
  return 0;
}'''
    tmp = os.path.join(ROOT, "build")
    os.makedirs(tmp, exist_ok=True)
    c = os.path.join(tmp, "layout_probe.c")
    exe = os.path.join(tmp, "layout_probe")
    open(c, "w").write(prog)
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), "-o", exe, c])
    vals = [int(v) for v in subprocess.check_output([exe]).split()]
    assert vals[0] == ctypes.sizeof(N.StConfig)
    assert vals[1] == ctypes.sizeof(N.StLayout)
    assert vals[2] == ctypes.sizeof(N.StStats)
    assert vals[3] == N.StConfig.capacity.offset
    assert vals[4] == N.StConfig.stream.offset
    assert vals[5] == N.StConfig.nccl_unique_id.offset
    assert vals[6] == N.StLayout.local_cells.offset


def test_config_default_and_abi_version(lib):
    from paper_2603_26691_b200 import _native as N
    c = N.StConfig()
    lib.st_config_default(ctypes.byref(c))
    assert c.abi_version == N.ST_ABI_VERSION == lib.st_abi_version()
    assert list(c.dims) == [16, 16, 16] and c.chunk_cells == 8 and c.rebin_interval == 1
    assert c.rho_f == 1.2 and c.nu_f == 1.5e-5 and c.rho_p == 1000.0


def test_init_validation_errors(lib):
    """Invalid configs are rejected before touching the GPU (ST_ERR_INVALID_ARG)."""
    from paper_2603_26691_b200 import _native as N
    c = N.StConfig()
    lib.st_config_default(ctypes.byref(c))
    c.rebin_interval = 0
    h = ctypes.c_void_p()
    assert lib.st_init(ctypes.byref(c), ctypes.byref(h)) == 1
    assert b"rebin_interval" in lib.st_last_error(None)
    lib.st_config_default(ctypes.byref(c))
    c.nranks = 4
    c.rank = 0
    c.dims[2] = 16          # 2 chunk planes < 4 ranks
    assert lib.st_init(ctypes.byref(c), ctypes.byref(h)) == 1


def test_no_cpu_fallback_without_gpu(lib):
    """Without a GPU the product path fails loudly (ST_ERR_CUDA), never computes on CPU."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2603_26691_b200 import Config, ScaleTrack, StError
    with pytest.raises(StError) as e:
        ScaleTrack(Config(capacity=10))
    assert e.value.status in (6, 8)


def test_binding_refuses_missing_library(tmp_path, monkeypatch):
    from paper_2603_26691_b200 import _native as N
    monkeypatch.setattr(N, "_lib", None)
    monkeypatch.setattr(N, "LIB_PATH", str(tmp_path / "missing.so"))
    with pytest.raises(ImportError):
        N.load()


def test_micro_config_layout_default_and_validation(lib):
    """st_micro_config: C layout == ctypes mirror; defaults are the C-30
    constants and match MicroConfig; invalid arguments fail before any device work."""
    from paper_2603_26691_b200 import _native as N
    from paper_2603_26691_b200.api import MicroConfig
    prog = r'''
#include <stdio.h>
#include <stddef.h>
#include "scaletrack.h"
int main(void){
  printf("%zu %zu %zu %zu %zu %d %d\n", sizeof(st_micro_config), offsetof(st_micro_config, D_v),
         offsetof(st_micro_config, device), offsetof(st_micro_config, stream),
         offsetof(st_micro_config, arithmetic), (int)ST_ARITH_FP64, (int)ST_ARITH_FP32);
  return 0;
}'''
    tmp = os.path.join(ROOT, "build")
    os.makedirs(tmp, exist_ok=True)
    c_src, exe = os.path.join(tmp, "micro_probe.c"), os.path.join(tmp, "micro_probe")
    open(c_src, "w").write(prog)
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), "-o", exe, c_src])
    vals = [int(v) for v in subprocess.check_output([exe]).split()]
    M = N.StMicroConfig
    assert vals == [ctypes.sizeof(M), M.D_v.offset, M.device.offset, M.stream.offset, M.arithmetic.offset,
                    N.ARITH_FP64, N.ARITH_FP32]
    c = M()
    lib.st_micro_config_default(ctypes.byref(c))
    py = MicroConfig().to_c()
    for f, _ in M._fields_:
        got, want = getattr(c, f), getattr(py, f)
        if hasattr(got, "_length_"):
            got, want = list(got), list(want)
        assert got == want, f
    nc = ctypes.c_int64(7)
    # n == 0 is a no-op even without a GPU; bad arguments are rejected first
    assert lib.st_micro_advance(ctypes.byref(c), 0, None, None, None, None, None, None, 1e-3, 1, None,
                                ctypes.byref(nc)) == 0 and nc.value == 0
    assert lib.st_micro_advance(ctypes.byref(c), 4, None, None, None, None, None, None, 1e-3, 1, None, None) == 1
    assert lib.st_micro_advance(ctypes.byref(c), 4, None, None, None, None, None, None, 0.0, 1, None, None) == 1
    bad = M()
    lib.st_micro_config_default(ctypes.byref(bad))
    bad.cell_size[1] = 0.0
    assert lib.st_micro_advance(ctypes.byref(bad), 0, None, None, None, None, None, None, 1e-3, 1, None, None) == 1
    bad.cell_size[1] = 1.0
    bad.arithmetic = 2                                # neither fp64 nor fp32
    assert lib.st_micro_advance(ctypes.byref(bad), 0, None, None, None, None, None, None, 1e-3, 1, None, None) == 1
    assert MicroConfig(arithmetic="fp32").to_c().arithmetic == N.ARITH_FP32
    with pytest.raises(ValueError):
        MicroConfig(arithmetic="bf16").to_c()
