"""Generic float64 operator kernels (csrc/generic.cu, bf_gx_* in include/bfgpu.h) against
numpy, one per operator kind of the reference's detail::eval_func (interpreter.hpp:263-299)
and the ScalarExpr programs of the three built-in examples (scalar_expr.hpp:66-87).
The graph walk that drives them is covered end to end by tests/test_cli.py (generic route)."""
import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ADD, MUL, ROW_SHIFT, ROW_SCALE = 0, 1, 2, 3
VAR, CONST, EADD, ESUB, EMUL, EDIV, EXP, SQRT, RECIP, SQUARE, SIGMOID = range(11)


@pytest.fixture(scope="module")
def env():
    import torch

    from paper_2505_07829_b200 import _lib

    return torch, _lib.lib()


def dev(torch, a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


def ptr(t):
    return ctypes.c_void_p(t.data_ptr())


def test_binary_and_row_ops(env):
    torch, lib = env
    rng = np.random.default_rng(1)
    a, b = rng.standard_normal((37, 53)), rng.standard_normal((37, 53))
    c = rng.standard_normal(37)
    A, B, C = dev(torch, a), dev(torch, b), dev(torch, c)
    out = torch.empty_like(A)
    for op, ref in [(ADD, a + b), (MUL, a * b)]:
        assert lib.bf_gx_binary(op, ptr(A), ptr(B), ptr(out), a.size, None) == 0
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy(), ref)
    for op, ref in [(ROW_SHIFT, a + c[:, None]), (ROW_SCALE, a * c[:, None])]:
        assert lib.bf_gx_row_op(op, ptr(A), ptr(C), ptr(out), 37, 53, None) == 0
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy(), ref)


def test_row_sum_dot_outer(env):
    torch, lib = env
    rng = np.random.default_rng(2)
    a, b = rng.standard_normal((70, 130)), rng.standard_normal((45, 130))
    u, v = rng.standard_normal(70), rng.standard_normal(45)
    A, B, U, V = dev(torch, a), dev(torch, b), dev(torch, u), dev(torch, v)
    rs = torch.empty(70, dtype=torch.float64, device="cuda")
    assert lib.bf_gx_row_sum(ptr(A), ptr(rs), 70, 130, None) == 0
    d = torch.empty(70, 45, dtype=torch.float64, device="cuda")
    assert lib.bf_gx_dot(ptr(A), ptr(B), ptr(d), 70, 45, 130, None) == 0
    o = torch.empty(70, 45, dtype=torch.float64, device="cuda")
    assert lib.bf_gx_outer(ptr(U), ptr(V), ptr(o), 70, 45, None) == 0
    torch.cuda.synchronize()
    np.testing.assert_allclose(rs.cpu().numpy(), a.sum(1), rtol=1e-13, atol=1e-13)
    np.testing.assert_allclose(d.cpu().numpy(), a @ b.T, rtol=1e-12, atol=1e-12)
    assert np.array_equal(o.cpu().numpy(), np.outer(u, v))


@pytest.mark.parametrize(
    "prog,consts,f",
    [
        ([VAR, VAR, SIGMOID, EMUL], None, lambda x: x / (1 + np.exp(-x))),  # swish (rms-swiglu)
        ([VAR, CONST, EDIV, CONST, EADD, SQRT, RECIP], [0, 4096.0, 0, 1e-5, 0, 0, 0],
         lambda x: 1 / np.sqrt(x / 4096.0 + 1e-5)),  # recip(sqrt(x / total(D) + eps))
        ([VAR, CONST, EDIV, EXP], [0, 11.3137, 0, 0], lambda x: np.exp(x / 11.3137)),  # attention exp
        ([CONST, VAR, CONST, EDIV, SQUARE, ESUB], [0.0, 0, 64.0, 0, 0, 0], lambda x: 0 - (x / 64.0) ** 2),
    ],
)
def test_elementwise_programs(env, prog, consts, f):
    torch, lib = env
    x = np.abs(np.random.default_rng(3).standard_normal(1000)) + 0.1
    X = dev(torch, x)
    out = torch.empty_like(X)
    ops = (ctypes.c_int8 * len(prog))(*prog)
    cst = (ctypes.c_double * len(prog))(*(consts or [0.0] * len(prog)))
    assert lib.bf_gx_elementwise(ops, cst, len(prog), ptr(X), ptr(out), x.size, None) == 0
    torch.cuda.synchronize()
    np.testing.assert_allclose(out.cpu().numpy(), f(x), rtol=1e-14, atol=1e-300)


def test_malformed_programs_rejected(env):
    torch, lib = env
    X = torch.zeros(4, dtype=torch.float64, device="cuda")
    for prog in ([EADD], [VAR, VAR], [VAR, 99]):
        ops = (ctypes.c_int8 * len(prog))(*prog)
        assert lib.bf_gx_elementwise(ops, None, len(prog), ptr(X), ptr(X), 4, None) == 1  # BF_ERR_INVALID_ARGUMENT
