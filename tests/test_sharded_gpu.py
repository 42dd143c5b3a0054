"""Multi-GPU paths behind the drop-in: bf_launch_sharded (one host thread,
N devices, optional all-gather) and the one-process-per-GPU launcher (torch.distributed).

The box has one GPU, so the N-device cases put several shards on device 0 (the sharding,
per-shard launches and the gather are the same code; the gather then takes the peer-copy
path), and the NCCL gather runs over a one-device communicator. Rows and heads are
independent in all three programs, so a sharded result must equal the single-launch result
bit for bit, and both must match the float64 oracle.
"""
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from helpers import assert_bf16_close, bf16_round

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


@pytest.fixture(scope="module")
def torch_mods():
    import torch

    from paper_2505_07829_b200 import launcher, ops

    return torch, ops, launcher


def _t(torch, a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda().bfloat16()


def _split(launcher, pattern, units, ngpu):
    return [launcher.shard_range(pattern, units, ngpu, g) for g in range(ngpu)]


@pytest.mark.parametrize("ngpu", [2, 3])
def test_ffn_sharded_gather_equals_single_launch(torch_mods, ngpu):
    torch, ops, launcher = torch_mods
    from oracle import cpu

    rng = np.random.default_rng(ngpu)
    M, D, F, N = 1000, 512, 1024, 512
    X = bf16_round(rng.standard_normal((M, D)))
    Wt, Vt = (bf16_round(rng.standard_normal((F, D)) / np.sqrt(D)) for _ in range(2))
    Ut = bf16_round(rng.standard_normal((N, F)) / np.sqrt(F))
    x, wt, vt, ut = (_t(torch, a) for a in (X, Wt, Vt, Ut))
    single = ops.rms_ffn_swiglu(x, wt, vt, ut)
    shards = []
    for lo, hi in _split(launcher, "rms_ffn_swiglu", M, ngpu):
        shards.append({"device": 0, "inputs": [x[lo:hi], wt, vt, ut],
                       "out": torch.empty(hi - lo, N, dtype=torch.bfloat16, device="cuda"),
                       "out_full": torch.empty(M, N, dtype=torch.bfloat16, device="cuda")})
    launcher.launch_sharded("rms_ffn_swiglu", shards, (M, D, F, N), gather=True)
    torch.cuda.synchronize()
    for sh in shards:
        assert torch.equal(sh["out_full"], single)
    assert_bf16_close(shards[0]["out_full"].double().cpu().numpy(), cpu.rms_ffn_swiglu(X, Wt, Vt, Ut),
                      f"K1 sharded x{ngpu} vs oracle")


def test_lnmm_and_attention_sharded(torch_mods):
    torch, ops, launcher = torch_mods
    from oracle import cpu

    rng = np.random.default_rng(9)
    M, K, N = 700, 256, 384
    X = bf16_round(rng.standard_normal((M, K)) * 2 + 1)
    Yt = bf16_round(rng.standard_normal((N, K)))
    x, yt = _t(torch, X), _t(torch, Yt)
    single = ops.layernorm_matmul(x, yt)
    shards = [{"device": 0, "inputs": [x[lo:hi], yt], "out": torch.empty(hi - lo, N, dtype=torch.bfloat16,
                                                                           device="cuda"),
               "out_full": torch.empty(M, N, dtype=torch.bfloat16, device="cuda")}
              for lo, hi in _split(launcher, "layernorm_matmul", M, 2)]
    launcher.launch_sharded("layernorm_matmul", shards, (M, K, N), gather=True)
    torch.cuda.synchronize()
    assert torch.equal(shards[1]["out_full"], single)
    assert_bf16_close(single.double().cpu().numpy(), cpu.layernorm_matmul(X, Yt), "K2 single")

    BH, S, Dh = 7, 384, 128
    Q, Kk = (bf16_round(rng.standard_normal((BH, S, Dh))) for _ in range(2))
    Vt = bf16_round(rng.standard_normal((BH, Dh, S)))
    q, k, v = _t(torch, Q), _t(torch, Kk), _t(torch, Vt)
    single = ops.attention(q, k, v)
    shards = [{"device": 0, "inputs": [q[lo:hi], k[lo:hi], v[lo:hi]],
               "out": torch.empty(hi - lo, S, Dh, dtype=torch.bfloat16, device="cuda"),
               "out_full": torch.empty(BH, S, Dh, dtype=torch.bfloat16, device="cuda")}
              for lo, hi in _split(launcher, "attention", BH, 3)]
    launcher.launch_sharded("attention", shards, (BH, S, S, Dh, Dh), gather=True)
    torch.cuda.synchronize()
    assert torch.equal(shards[2]["out_full"], single)


def test_nccl_gather_one_device(torch_mods):
    """The NCCL all-gather-v path (dlopen'd libnccl, single-process communicator) on one device."""
    torch, ops, launcher = torch_mods
    from paper_2505_07829_b200 import _lib

    assert _lib.lib().bf_nccl_version() > 0
    rng = np.random.default_rng(3)
    M, K, N = 300, 128, 256
    x, yt = _t(torch, rng.standard_normal((M, K))), _t(torch, rng.standard_normal((N, K)))
    single = ops.layernorm_matmul(x, yt)
    sh = {"device": 0, "inputs": [x, yt], "out": torch.empty(M, N, dtype=torch.bfloat16, device="cuda"),
          "out_full": torch.zeros(M, N, dtype=torch.bfloat16, device="cuda")}
    os.environ["BFGPU_GATHER"] = "nccl"
    try:
        launcher.launch_sharded("layernorm_matmul", [sh], (M, K, N), gather=True)
        torch.cuda.synchronize()
    finally:
        del os.environ["BFGPU_GATHER"]
    assert torch.equal(sh["out_full"], single)


WORKER = r"""
import os, sys, numpy as np, torch, torch.distributed as dist
sys.path.insert(0, {root!r}); sys.path.insert(0, {tests!r})
from paper_2505_07829_b200 import ops
from paper_2505_07829_b200.launcher import shard, gather_rows
from helpers import assert_bf16_close, bf16_round
dist.init_process_group("gloo", init_method="tcp://127.0.0.1:{port}", rank=int(sys.argv[1]), world_size=2)
rank = dist.get_rank()
rng = np.random.default_rng(0)
M, D, F, N = 900, 256, 512, 256
X = bf16_round(rng.standard_normal((M, D))); Wt = bf16_round(rng.standard_normal((F, D)) / 16)
Vt = bf16_round(rng.standard_normal((F, D)) / 16); Ut = bf16_round(rng.standard_normal((N, F)) / 16)
shards = [shard(M, r, 2, 128) for r in range(2)]
s = shards[rank]
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda().bfloat16()
O = ops.rms_ffn_swiglu(t(X[s.start:s.stop]), t(Wt), t(Vt), t(Ut))
torch.cuda.synchronize()
full = gather_rows(O.float().cpu(), shards)   # gloo all-gather of the row shards
# K2: token rows, Yt replicated
Mx, K2, N2 = 700, 256, 384
Xl = bf16_round(rng.standard_normal((Mx, K2)) * 2 + 1); Yt = bf16_round(rng.standard_normal((N2, K2)))
lsh = [shard(Mx, r, 2, 128) for r in range(2)]
Ol = ops.layernorm_matmul(t(Xl[lsh[rank].start:lsh[rank].stop]), t(Yt))
torch.cuda.synchronize()
full_l = gather_rows(Ol.float().cpu(), lsh)
# K3: heads
BH, S, Dh = 5, 256, 128
Q = bf16_round(rng.standard_normal((BH, S, Dh))); Kk = bf16_round(rng.standard_normal((BH, S, Dh)))
Va = bf16_round(rng.standard_normal((BH, Dh, S)))
hsh = [shard(BH, r, 2, 1) for r in range(2)]
h = hsh[rank]
Oa = ops.attention(t(Q[h.start:h.stop]), t(Kk[h.start:h.stop]), t(Va[h.start:h.stop]))
torch.cuda.synchronize()
full_a = gather_rows(Oa.float().cpu(), hsh)
if rank == 0:
    from oracle import cpu
    assert_bf16_close(full.double().numpy(), cpu.rms_ffn_swiglu(X, Wt, Vt, Ut), "K1 2-rank gather vs oracle")
    assert_bf16_close(full_l.double().numpy(), cpu.layernorm_matmul(Xl, Yt), "K2 2-rank gather vs oracle")
    assert_bf16_close(full_a.double().numpy(), cpu.attention_safe(Q, Kk, Va), "K3 2-rank head gather vs oracle")
    print("ok", full.shape)
dist.barrier()
dist.destroy_process_group()
"""


def test_two_process_row_shards_gloo():
    """World size 2, one process per shard (both on cuda:0 here), each running K1 and K2 on its
    rows and K3 on its heads; the gathered outputs match the oracle."""
    import socket

    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    code = WORKER.format(root=str(ROOT), tests=str(ROOT / "tests"), port=port)
    procs = [subprocess.Popen([sys.executable, "-c", code, str(r)], stdout=subprocess.PIPE, stderr=subprocess.PIPE,
                              text=True) for r in range(2)]
    outs = [p.communicate(timeout=600) for p in procs]
    for p, (o, e) in zip(procs, outs):
        assert p.returncode == 0, f"{o}\n{e[-3000:]}"
    assert "ok" in outs[0][0]
