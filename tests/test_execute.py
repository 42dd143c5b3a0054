"""The drop-in boundary at the reference's own C++ API: bfgpu::execute has the
signature of blockfuse::execute (interpreter.hpp:478-487). These tests drive it
through tests/cpp/libbfx_selftest.so (built by host/Makefile from the
unmodified reference headers) on the reference's own programs and inputs.

CPU part: recognition of every fusion snapshot (and rejection of anything
else) needs no device. GPU part: the adapter's outputs vs the reference CPU
executor on the same program, inputs and binding, mirroring the reference's
acceptance criteria 2-4 (tests/acceptance.cpp:114-201) at tensor-core sizes.
"""
import ctypes
from pathlib import Path

import pytest

from helpers import BF16_REL_TOL, F32_REL_TOL

LIB = Path(__file__).resolve().parent / "cpp" / "libbfx_selftest.so"
ATTN, LNMM, FFN = 0, 1, 2
SNAPSHOTS = {ATTN: 2, LNMM: 2, FFN: 3}  # acceptance.cpp criteria 1, 3, 4

if not LIB.exists():
    pytest.skip("adapter test harness not built (make -C host)", allow_module_level=True)


@pytest.fixture(scope="module")
def lib():
    l = ctypes.CDLL(str(LIB))
    l.bfx_recognize.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.POINTER(ctypes.c_int),
                                ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_double), ctypes.c_char_p,
                                ctypes.c_int]
    l.bfx_compare.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_char_p, ctypes.c_int, ctypes.c_ulonglong,
                              ctypes.c_double, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double),
                              ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int), ctypes.c_char_p, ctypes.c_int]
    return l


def recognize(lib, which, snap, eps=0.0):
    p, s, e = ctypes.c_int(), ctypes.c_int(), ctypes.c_double()
    msg = ctypes.create_string_buffer(512)
    rc = lib.bfx_recognize(which, snap, eps, ctypes.byref(p), ctypes.byref(s), ctypes.byref(e), msg, 512)
    return rc, p.value, s.value, e.value, msg.value.decode()


@pytest.mark.parametrize("which", [ATTN, LNMM, FFN])
def test_every_snapshot_is_recognized(lib, which):
    for snap in range(SNAPSHOTS[which]):
        rc, pat, s, _, msg = recognize(lib, which, snap)
        assert rc == 0, msg
        assert s == snap
        # pattern enum: RmsFfnSwiglu=0, LayerNormMatMul=1, Attention=2
        assert pat == {ATTN: 2, LNMM: 1, FFN: 0}[which]


def test_materializing_snapshots_flagged(lib):
    # K1 snapshot 0 keeps H buffered and attention snapshot 0 keeps P buffered
    assert recognize(lib, FFN, 0)[4] == "materializes"
    assert recognize(lib, ATTN, 0)[4] == "materializes"
    assert recognize(lib, FFN, 2)[4] == "fused"
    assert recognize(lib, LNMM, 1)[4] == "fused"


@pytest.mark.parametrize("which", [ATTN, LNMM, FFN])
def test_unfused_program_is_rejected(lib, which):
    rc, *_, msg = recognize(lib, which, -2)
    assert rc != 0
    assert "no CPU fallback" in msg


def test_rmsnorm_epsilon_recovered(lib):
    rc, pat, snap, eps, msg = recognize(lib, FFN, -1, eps=1e-5)
    assert rc == 0, msg
    assert eps == 1e-5


def compare(lib, which, snap, binding, precision, seed, eps=0.0):
    rel, norm = ctypes.c_double(), ctypes.c_double()
    p, s = ctypes.c_int(), ctypes.c_int()
    msg = ctypes.create_string_buffer(1024)
    rc = lib.bfx_compare(which, snap, binding.encode(), precision, seed, eps, ctypes.byref(rel), ctypes.byref(norm),
                         ctypes.byref(p), ctypes.byref(s), msg, 1024)
    return rc, rel.value, norm.value, msg.value.decode()


CASES = [
    # acceptance-suite bindings (count 2, len 4) run in fp32 mode: any shape is legal there
    (FFN, "D=2x4,K=2x4,M=2x4,N=2x4", 1, 3000),
    (LNMM, "K=2x4,M=2x4,N=2x4", 1, 2000),
    (ATTN, "D=2x4,L=2x4,M=2x4,N=2x4", 1, 1000),
    # asymmetric binding of test_engine.cpp:221-238
    (FFN, "D=1x4,K=4x2,M=3x2,N=2x3", 1, 6),
    (ATTN, "D=1x4,L=2x2,M=3x2,N=2x3", 1, 5),
    # tensor-core sizes, bf16 mode
    (FFN, "D=2x128,K=3x128,M=3x64,N=2x128", 0, 31),
    (LNMM, "K=2x128,M=3x64,N=3x128", 0, 32),
    (ATTN, "D=1x128,L=1x128,M=2x128,N=3x128", 0, 33),
]


@pytest.mark.gpu
@pytest.mark.parametrize("which,binding,precision,seed", CASES)
def test_adapter_matches_reference_executor(lib, which, binding, precision, seed):
    for snap in range(SNAPSHOTS[which]):
        rc, rel, norm, msg = compare(lib, which, snap, binding, precision, seed)
        assert rc == 0, msg
        tol = F32_REL_TOL if precision == 1 else BF16_REL_TOL
        assert rel <= tol, f"snapshot {snap}: max|d|/max|ref| = {rel:.3e}"


@pytest.mark.gpu
def test_adapter_eps(lib):
    rc, rel, norm, msg = compare(lib, FFN, -1, "D=2x128,K=2x128,M=2x128,N=1x128", 1, 9, eps=1e-3)
    assert rc == 0, msg
    assert rel <= F32_REL_TOL


# The reference's input errors (eval_graph's Input case, interpreter.hpp:386-403, and
# DimBinding, :49-58): the drop-in raises the same blockfuse::Error messages, before any device
# work, so this runs on the CPU. kind 0: an input missing; 1: one row too many; 2: one column
# too many; 3: dimension M unbound.
@pytest.mark.parametrize("which", [ATTN, LNMM, FFN])
@pytest.mark.parametrize("kind", [0, 1, 2, 3])
def test_input_errors_match_reference(lib, which, kind):
    lib.bfx_error_case.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_char_p, ctypes.c_char_p, ctypes.c_char_p,
                                   ctypes.c_int]
    binding = {ATTN: b"M=2x4,N=2x4,D=2x4,L=2x4", LNMM: b"M=2x4,N=2x4,K=2x4", FFN: b"M=2x4,N=2x4,D=2x4,K=2x4"}[which]
    ref, ours = ctypes.create_string_buffer(512), ctypes.create_string_buffer(512)
    threw = lib.bfx_error_case(which, kind, binding, ref, ours, 512)
    assert threw == 2, (ref.value, ours.value)
    assert ours.value == ref.value
    expect = {0: b"missing input matrix", 1: b"row count does not match binding",
              2: b"column count does not match binding", 3: b"unbound dimension M"}[kind]
    assert expect in ref.value


def test_host_conversions_are_bit_exact(lib):
    """The adapter's AVX2 fp64 -> bf16 narrowing and bf16 -> fp64 widening (host/convert.hpp) equal
    their scalar forms bit for bit: ties, subnormals, infinities, overflow to inf, NaN."""
    lib.bfx_conversion_check.argtypes = [ctypes.c_long, ctypes.c_ulonglong]
    lib.bfx_conversion_check.restype = ctypes.c_long
    for n, seed in ((1 << 20, 1), (1003, 2), (7, 3)):
        assert lib.bfx_conversion_check(n, seed) == 0
