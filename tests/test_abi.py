"""C-ABI library: loads without a GPU, exports every symbol of include/lightgp.h,
host-only entry points behave, and the kernel-tree JIT compiles for sm_100a
(NVRTC runs on the host) without register spills in the hot kernel."""

import ctypes as C
import os
import re

import numpy as np
import pytest

from conftest import ROOT
from paper_2605_17898_b200 import _lib
import paper_2605_17898_b200 as G


def header_symbols():
    text = open(os.path.join(ROOT, "include", "lightgp.h")).read()
    return sorted(set(re.findall(r"^(?:int|const char\*)\s+(lgp_\w+)\(", text, re.M)))


def test_library_loads_and_exports_header():
    lib = _lib.lib()
    syms = header_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_lib.exported_symbols())
    assert lib.lgp_abi_version() == 1


def test_partition():
    lib = _lib.lib()
    r0, r1 = C.c_int64(), C.c_int64()
    n = 100_003
    seen = []
    for w in (1, 2, 3, 8):
        cover = 0
        for r in range(w):
            _lib.check(lib.lgp_partition(n, w, r, C.byref(r0), C.byref(r1)))
            assert r1.value - r0.value <= -(-n // w)
            cover += r1.value - r0.value
            seen.append((r0.value, r1.value))
        assert cover == n
    with pytest.raises(ValueError):
        _lib.check(lib.lgp_partition(10, 2, 2, C.byref(r0), C.byref(r1)))


def test_kernel_compile_validation():
    with pytest.raises(ValueError):
        _lib.KernelProgram([0], [-1.0])  # nonpositive lengthscale
    with pytest.raises(ValueError):
        _lib.KernelProgram([7, 0], [1.0])  # Sum missing a child
    with pytest.raises(ValueError):
        _lib.KernelProgram([0, 0], [1.0, 1.0])  # trailing node
    with pytest.raises(ValueError):
        _lib.KernelProgram([42], [1.0])  # unknown kind
    p = _lib.KernelProgram([6, 0], [2.0, 0.5])
    assert "lgp_matvec" in p.source(d=3)


JIT_CASES = [
    ("(rbf 0.5)", 8, 16), ("(rbf 0.5)", 8, 1), ("(rbf 0.2)", 1, 1), ("(matern52 0.5)", 4, 1),
    ("(+ (scale 1.0 (rbf 0.5)) (scale 1.0 (periodic 1.0 1.0)))", 2, 16),
    ("(matern32 0.5)", 8, 8), ("(+ (scale 2.0 (matern32 0.4)) (linear 0.5))", 3, 1),
]


@pytest.mark.parametrize("expr,d,t", JIT_CASES)
def test_jit_compiles_without_spills(expr, d, t):
    log = G.kernels.program(G.parse_kernel(expr)).jit(d, t)
    # ptxas -v reports one block per kernel; the matvec kernel must not spill
    blocks = re.split(r"Compiling entry function", log)
    mv = [b for b in blocks if "'lgp_matvec'" in b]
    assert mv, log
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", mv[0])
    assert m and m.group(1) == "0" and m.group(2) == "0", mv[0]
    regs = int(re.search(r"Used (\d+) registers", mv[0]).group(1))
    assert regs <= 255


def test_generated_source_mentions_tree():
    # cfg3's tree at t = 16: tensor-core kernel with staged Periodic features
    src = G.kernels.program(G.parse_kernel("(+ (scale 1.0 (rbf 0.5)) (scale 1.0 (periodic 1.0 1.0)))")).source(2, 16)
    assert "lgp_matvec_tc" in src and "lgp_tc_prep_feat" in src and "sincos" in src
    assert "#define LGP_TC_PF 4" in src
    # a Matern-1/2 tree stays on the SIMT kernel
    src = G.kernels.program(G.parse_kernel("(+ (scale 1.0 (matern12 0.5)) (periodic 1.0 1.0))")).source(2, 16)
    assert "lgp_ex2" in src and "cp.async.bulk" in src and "#define LGP_TB 16" in src
    assert "lgp_matvec_tc" not in src


def test_no_gpu_fails_loudly():
    n = C.c_int()
    _lib.check(_lib.lib().lgp_device_count(C.byref(n)))
    if n.value > 0:
        pytest.skip("GPU present")
    with pytest.raises(G.MiniGpError, match="no CUDA device"):
        _lib.Context(0)


def test_tensor_core_jit_compiles_with_tcgen05():
    import glob
    import subprocess

    log = G.kernels.program(G.parse_kernel("(rbf 0.5)")).jit(8, 16)
    assert "[tensor-core module]" in log and "'lgp_matvec_tc'" in log
    tc = log.split("[tensor-core module]")[1]
    m = re.search(r"'lgp_matvec_tc'.*?(\d+) bytes spill stores", tc, re.S)
    # 12 warps cap the kernel at 168 registers; ptxas parks a couple of
    # loop-invariant values on the stack (<= 16 bytes), nothing more
    assert m and int(m.group(1)) <= 16
    # the cached cubin's SASS proves tcgen05 MMA, TMEM ld/st and TMA bulk copies
    src = G.kernels.program(G.parse_kernel("(rbf 0.5)")).source(8, 16)
    cache = os.path.join(ROOT, "paper_2605_17898_b200", "_lib", "jit_cache")
    cubins = [p for p in glob.glob(os.path.join(cache, "*.cu"))
              if open(p).read().strip() == src.strip()]
    assert cubins, "tensor-core module not in the JIT cache"
    sass = subprocess.run(["cuobjdump", "-sass", cubins[0][:-3] + ".cubin"], capture_output=True,
                          text=True).stdout
    for mnemonic in ("UTCHMMA", "LDTM", "STTM", "UBLKCP", "MUFU.EX2", "FHFMA"):
        assert mnemonic in sass, mnemonic
