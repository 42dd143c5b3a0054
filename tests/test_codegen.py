"""The block-program compiler (host/bfgpu_codegen.cpp): programs the fused kernels do not
cover are compiled to CUDA, one kernel per top-level operator, and built with NVRTC for
sm_100a (bf_jit_compile). The reference interprets them (eval_graph -> eval_map ->
eval_func, interpreter.hpp:263-472).

CPU: the generated source of every program of the fusion driver (the unfused lower()
program and every snapshot of the three examples) at the acceptance-suite and asymmetric
bindings (tests/acceptance.cpp:114-201, tests/test_engine.cpp:221-238) compiles with NVRTC,
with one kernel per top-level operator (metrics.hpp kernel_count) and the safety pass's
significand/exponent pairs where the program exponentiates. GPU: results against the
reference CPU interpreter live in tests/test_cli.py and test_execute.py; the extreme-logit
case here.
"""
import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
LIB = ROOT / "tests" / "cpp" / "libbfx_selftest.so"
ATTN, LNMM, FFN = 0, 1, 2
SNAPSHOTS = {ATTN: 2, LNMM: 2, FFN: 3}
BINDINGS = {
    ATTN: ["M=2x4,N=2x4,D=2x4,L=2x4", "M=3x2,N=2x3,D=1x4,L=2x2"],
    LNMM: ["M=2x4,N=2x4,K=2x4", "M=3x2,N=2x3,K=4x2"],
    FFN: ["M=2x4,N=2x4,D=2x4,K=2x4", "M=3x2,N=2x3,D=1x4,K=4x2"],
}


def top_level_operators(which, snap):
    """The reference's kernel_count (metrics.hpp): one generated kernel per top-level operator.
    From the reference build when present (oracle/_ref), else its known values."""
    try:
        from oracle import refexec as R

        if R.available():
            return R.program_stats({ATTN: R.ATTENTION, LNMM: R.LAYERNORM_MATMUL, FFN: R.RMS_FFN_SWIGLU}[which],
                                   R.UNFUSED if snap == -2 else snap)["kernels"]
    except Exception:
        pass
    return {ATTN: 7, LNMM: 8, FFN: 9}[which] if snap == -2 else 1

if not LIB.exists():
    pytest.skip("adapter test harness not built (make -C host)", allow_module_level=True)


@pytest.fixture(scope="module")
def libs():
    from paper_2505_07829_b200 import _lib

    l = ctypes.CDLL(str(LIB))
    l.bfx_generic_source.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_char_p, ctypes.c_char_p, ctypes.c_long,
                                     ctypes.c_char_p, ctypes.c_int]
    return l, _lib.lib()


def source(l, which, snap, binding):
    buf = ctypes.create_string_buffer(1 << 22)
    msg = ctypes.create_string_buffer(2048)
    rc = l.bfx_generic_source(which, snap, binding.encode(), buf, len(buf), msg, len(msg))
    assert rc == 0, msg.value.decode()
    return buf.value.decode()


@pytest.mark.parametrize("which", [ATTN, LNMM, FFN])
def test_generated_source_compiles_for_every_program(libs, which):
    l, bf = libs
    for binding in BINDINGS[which]:
        for snap in [-2] + list(range(SNAPSHOTS[which])):
            src = source(l, which, snap, binding)
            kernels = re.findall(r'extern "C" __global__ void __launch_bounds__\(256\) (\w+)', src)
            assert len(kernels) == top_level_operators(which, snap), (snap, kernels)
            log = ctypes.create_string_buffer(1 << 16)
            rc = bf.bf_jit_check(src.encode(), log, len(log))
            assert rc == 0, f"{which} snap {snap} {binding}: {bf.bf_last_error().decode()[:3000]}"


def test_safety_pass_rewrites_exponentials(libs):
    """The attention programs exponentiate: the compiled code keeps significand/exponent pairs
    (row maxima subtracted before exp, rebased accumulation) instead of the reference's plain exp."""
    l, _ = libs
    for snap in range(SNAPSHOTS[ATTN]):
        src = source(l, ATTN, snap, BINDINGS[ATTN][0])
        body = src[src.index('extern "C"'):]
        assert "se_add(" in body and "BF_NEG_INF" in body and "se_materialize(" in body
    # the layernorm program has no exponential: no pairs
    body = source(l, LNMM, 1, BINDINGS[LNMM][0])
    assert "se_add(" not in body[body.index('extern "C"'):]


@pytest.mark.gpu
def test_extreme_logits_finite_only_with_safety_pass():
    """The reference's fused attention program exponentiates without subtracting a maximum
    (the unsafe exp of lowering.hpp's softmax). With logits beyond exp's range the compiled
    program stays finite and equals safe_attention_rows (tests/test_safe_numerics.cpp:204-209);
    with the pass disabled (BFGPU_SAFE=0) it overflows like the interpreter."""
    import os
    import subprocess
    import sys

    code = r"""
import ctypes, sys, numpy as np
sys.path.insert(0, %r)
from oracle import refexec as R
L = ctypes.CDLL(%r)
L.bfx_attention_generic.argtypes = [ctypes.c_int, ctypes.c_char_p, ctypes.c_double, ctypes.POINTER(ctypes.c_double),
                                    ctypes.POINTER(ctypes.c_double), ctypes.c_char_p, ctypes.c_int]
got, safe = ctypes.c_double(), ctypes.c_double()
msg = ctypes.create_string_buffer(1024)
rc = L.bfx_attention_generic(1, b"M=2x4,N=3x4,D=2x4,L=2x4", 400.0, ctypes.byref(got), ctypes.byref(safe), msg, 1024)
print(rc, got.value, safe.value, msg.value.decode())
"""
    for env, finite in [("1", True), ("0", False)]:
        r = subprocess.run([sys.executable, "-c", code % (str(ROOT), str(LIB))], capture_output=True, text=True,
                           env={**os.environ, "BFGPU_SAFE": env, "BFGPU_QUIET": "1"}, timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        rc, err, safe_err, msg = r.stdout.split(maxsplit=3)
        assert rc == "0", msg
        if finite:
            assert float(err) < 1e-10, r.stdout  # max rel. error vs safe_attention_rows
        else:
            assert err in ("nan", "inf") or float(err) > 1e-3, r.stdout


# The reference interpreter's own test programs (tests/test_interpreter.cpp:46-178, via
# tests/test_util.hpp) through the compiler, against blockfuse::execute on the same inputs.
INTERP_CASES = {0: "identity elementwise", 1: "row sums: map over column blocks + fold",
                2: "relu_matmul unfused", 3: "relu_matmul fused by hand", 4: "relu_matmul, driver's final snapshot",
                5: "top-level Misc node with a host executor", 6: "map iteration order (permuted M blocks)"}


@pytest.mark.gpu
@pytest.mark.parametrize("case", sorted(INTERP_CASES))
def test_reference_interpreter_programs_on_the_compiler(libs, case):
    l, _ = libs
    l.bfx_interp_case.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_double), ctypes.c_char_p, ctypes.c_int]
    err = ctypes.c_double()
    msg = ctypes.create_string_buffer(1024)
    rc = l.bfx_interp_case(case, ctypes.byref(err), msg, 1024)
    assert rc == 0, f"{INTERP_CASES[case]}: {msg.value.decode()}"
    assert err.value <= 1e-12, f"{INTERP_CASES[case]}: max rel err {err.value:.3e}"
