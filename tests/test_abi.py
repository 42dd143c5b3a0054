"""CPU tests of the drop-in boundary: libbfgpu.so loads, exports exactly what
include/bfgpu.h declares, validates arguments, and fails loudly (never falls
back to the CPU) when no sm_100 device is present."""
import ctypes
import re
from pathlib import Path

import pytest

from paper_2505_07829_b200 import _lib

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    text = (ROOT / "include" / "bfgpu.h").read_text()
    return sorted(set(re.findall(r"BF_API\s+[\w\s\*]+?\b(bf_\w+)\s*\(", text)))


def test_header_and_binding_agree():
    assert declared_symbols() == sorted(_lib.EXPORTED)


def test_library_exports_every_declared_symbol():
    lib = _lib.lib()
    for name in declared_symbols():
        assert hasattr(lib, name), name


def test_introspection_without_gpu():
    lib = _lib.lib()
    assert lib.bf_version() >= 1
    assert lib.bf_kernel_launches() >= 0
    assert lib.bf_rms_ffn_swiglu_workspace_bytes(8192, 4096, 14336, 4096, _lib.BF_DTYPE_BF16, 0) >= 8192 * 14336 * 2
    assert lib.bf_rms_ffn_swiglu_workspace_bytes(0, 1, 1, 1, 0, 0) == 0


def test_null_pointers_rejected():
    lib = _lib.lib()
    rc = lib.bf_rms_ffn_swiglu(None, None, None, None, None, 1, 8, 8, 8, 0, 0.0, 0, None, 0, None)
    assert rc == _lib.BF_ERR_INVALID_ARGUMENT
    assert b"null" in lib.bf_last_error()


def test_compute_fails_loudly_without_sm100():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    lib = _lib.lib()
    dummy = ctypes.c_void_p(16)
    rc = lib.bf_layernorm_matmul(dummy, dummy, dummy, 128, 64, 64, 0, 0.0, dummy, 1 << 20, None)
    assert rc in (_lib.BF_ERR_CUDA, _lib.BF_ERR_UNSUPPORTED)
    assert lib.bf_last_error()
    rc = lib.bf_attention(dummy, dummy, dummy, dummy, 1, 128, 128, 128, 128, 0, 0.0, None)
    assert rc in (_lib.BF_ERR_CUDA, _lib.BF_ERR_UNSUPPORTED)


def test_ops_reject_cpu_tensors():
    import torch

    from paper_2505_07829_b200 import ops

    x = torch.zeros(4, 8, dtype=torch.bfloat16)
    with pytest.raises(ValueError, match="CUDA"):
        ops.layernorm_matmul(x, x)


def test_sass_contains_tcgen05_and_tma():
    """The built kernels are Blackwell-native: UTC*MMA (tcgen05.mma), LDTM/STTM
    (tcgen05.ld/st) and UTMALDG/UTMASTG (TMA) in the sm_100a SASS."""
    import shutil
    import subprocess

    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not Path(cuobjdump).exists():
        pytest.skip("cuobjdump not available")
    sass = subprocess.run([cuobjdump, "-sass", str(_lib.lib_path())], capture_output=True, text=True).stdout
    assert "sm_100a" in sass
    for mnem in ("UTCHMMA", "LDTM", "STTM", "UTMALDG", "UTMASTG"):
        assert mnem in sass, mnem
    assert "HMMA" not in sass.replace("UTCHMMA", "")


def test_misaligned_bf16_buffers_rejected():
    """Checked before any device query, so the error is the same with or without a GPU."""
    lib = _lib.lib()
    ok, bad = 1 << 20, (1 << 20) + 8
    rc = lib.bf_layernorm_matmul(bad, ok, ok, 128, 64, 64, _lib.BF_DTYPE_BF16, 0.0, ok, 1 << 20, None)
    assert rc == _lib.BF_ERR_INVALID_ARGUMENT
    assert b"16-byte aligned" in lib.bf_last_error()
    rc = lib.bf_attention(ok, ok, ok, bad, 1, 128, 128, 128, 128, _lib.BF_DTYPE_BF16, 0.0, None)
    assert rc == _lib.BF_ERR_INVALID_ARGUMENT
    rc = lib.bf_rms_ffn_swiglu(ok, ok, bad, ok, ok, 8, 8, 8, 8, _lib.BF_DTYPE_BF16, 0.0, 0, ok, 1 << 20, None)
    assert rc == _lib.BF_ERR_INVALID_ARGUMENT
