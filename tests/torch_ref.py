"""fp32 torch references of the three fused programs, computed on the GPU (TF32 off).

They state the dense forms of the reference's `ref::` oracles
(interpreter.hpp:543-559) in fp32 from the same bf16 inputs the kernels see,
so full-shape outputs (every row, every head) can be checked without moving
them to the host. The float64 oracle (oracle/bf_oracle.c, pinned to the
reference build) checks stratified rows of the same outputs, which pins these.
Each generator yields (row slice, reference chunk).
"""
from __future__ import annotations

import torch


def _no_tf32():
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.allow_tf32 = False


def rms_ffn_swiglu_chunks(X, Wt, Vt, Ut, eps: float = 0.0, chunk: int = 2048):
    """ref::rms_ffn_swiglu (interpreter.hpp:553-559) by row chunks."""
    _no_tf32()
    Wf, Vf, Uf = Wt.float(), Vt.float(), Ut.float()
    for a in range(0, X.shape[0], chunk):
        x = X[a:a + chunk].float()
        r = torch.rsqrt(x.pow(2).mean(dim=1, keepdim=True) + eps)
        g = (x @ Wf.T) * r
        u = (x @ Vf.T) * r
        h = torch.nn.functional.silu(g) * u
        yield slice(a, a + x.shape[0]), h @ Uf.T
    del Wf, Vf, Uf


def layernorm_matmul_chunks(X, Yt, chunk: int = 8192):
    """ref::layernorm_matmul (interpreter.hpp:549-551): layernorm without eps/gamma/beta, then X Yt^T."""
    _no_tf32()
    Yf = Yt.float()
    for a in range(0, X.shape[0], chunk):
        x = X[a:a + chunk].float()
        mu = x.mean(dim=1, keepdim=True)
        xc = x - mu
        xn = xc * torch.rsqrt(xc.pow(2).mean(dim=1, keepdim=True))
        yield slice(a, a + x.shape[0]), xn @ Yf.T


def attention_chunks(Q, K, Vt, scale: float | None = None, heads: int = 16):
    """ref::attention (interpreter.hpp:543-547) per head: softmax(scale Q K^T) V with V = Vt^T.
    The max-subtracted softmax equals safe_attention_rows (safe_numerics.hpp:147-175)."""
    _no_tf32()
    lead = Q.shape[:-2]
    q = Q.reshape(-1, *Q.shape[-2:])
    k = K.reshape(-1, *K.shape[-2:])
    v = Vt.reshape(-1, *Vt.shape[-2:])
    s = scale if scale is not None else Q.shape[-1] ** -0.5
    for a in range(0, q.shape[0], heads):
        sc = torch.bmm(q[a:a + heads].float(), k[a:a + heads].float().transpose(1, 2)) * s
        p = torch.softmax(sc, dim=-1)
        yield slice(a, a + sc.shape[0]), torch.bmm(p, v[a:a + heads].float().transpose(1, 2))
    del lead
