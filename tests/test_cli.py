"""Program-file front door (tools/bfgpu_cli.cpp).

The reference workflow `blockfuse examples X | blockfuse lower | blockfuse fuse`
(tools/blockfuse_main.cpp:139-181) writes "blockfuse-program" v1 JSON files
(bf/serialize.hpp:305-366). tests/golden/programs/ holds those files for the three
built-in programs, written by the reference's own fuse() and serializer
(`bfgpu-cli snapshots`, regenerated and compared below). The CLI feeds them to the
drop-in bfgpu::execute; exit codes follow the reference CLI (0 ok, 1 error,
2 inequivalent, tools/blockfuse_main.cpp:216-236).

CPU: recognition of every snapshot, rejection of the unfused programs and of
malformed files, byte-identical regeneration. GPU: `verify` against the reference
CPU interpreter at the acceptance-suite bindings (fp32 mode) and at tensor-core
sizes (bf16 mode), and `run`.
"""
import json
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
CLI = ROOT / "paper_2505_07829_b200" / "lib" / "bfgpu-cli"
PROGRAMS = Path(__file__).resolve().parent / "golden" / "programs"
EXAMPLES = {"attention": ("attention", 2), "layernorm-matmul": ("layernorm_matmul", 2),
            "rms-swiglu": ("rms_ffn_swiglu", 3)}

if not CLI.exists():
    pytest.skip("bfgpu-cli not built (make -C host)", allow_module_level=True)


def cli(*args, check=None):
    r = subprocess.run([str(CLI), *map(str, args)], capture_output=True, text=True, timeout=600)
    if check is not None:
        assert r.returncode == check, f"rc={r.returncode}\nstdout: {r.stdout}\nstderr: {r.stderr}"
    return r


@pytest.mark.parametrize("example", sorted(EXAMPLES))
def test_every_snapshot_file_is_recognized(example):
    pattern, count = EXAMPLES[example]
    for k in range(1, count + 1):
        r = cli("recognize", PROGRAMS / example / f"snapshot_{k}.json", check=0)
        got = json.loads(r.stdout)
        assert got["pattern"] == pattern and got["snapshot"] == k - 1 and got["output"] == "O"
    # the first attention and rms snapshots keep an internal buffered edge (P, H)
    first = json.loads(cli("recognize", PROGRAMS / example / "snapshot_1.json", check=0).stdout)
    assert first["materializes_intermediate"] == (example != "layernorm-matmul")


@pytest.mark.parametrize("example", sorted(EXAMPLES))
def test_unfused_program_file_is_rejected(example):
    r = cli("recognize", PROGRAMS / example / "lowered.json", check=1)
    assert "no CPU fallback" in r.stderr


def test_malformed_files_are_errors(tmp_path):
    bad = tmp_path / "bad.json"
    bad.write_text("{not json")
    assert "syntax error" in cli("recognize", bad, check=1).stderr
    other = tmp_path / "other.json"
    other.write_text(json.dumps({"format": "something-else"}))
    assert "not a program file" in cli("recognize", other, check=1).stderr
    assert "cannot open" in cli("recognize", tmp_path / "missing.json", check=1).stderr
    assert cli("frobnicate", check=1).returncode == 1


@pytest.mark.parametrize("example", sorted(EXAMPLES))
def test_fixtures_regenerate_identically(example, tmp_path):
    """The committed program files are exactly what the reference's fuse() emits."""
    cli("snapshots", example, "--out-dir", tmp_path, check=0)
    for f in sorted((PROGRAMS / example).glob("*.json")):
        assert (tmp_path / f.name).read_text() == f.read_text(), f.name


# dims/len per example: the acceptance bindings (count 2, len 4; tests/acceptance.cpp:114-201)
# in fp32 mode, and tensor-core sizes in bf16 mode
VERIFY = [
    ("attention", "M=2,N=2,D=2,L=2", "4x4", "", "f32"),
    ("layernorm-matmul", "M=2,N=2,K=2", "4x4", "", "f32"),
    ("rms-swiglu", "M=2,N=2,K=2,D=2", "4x4", "", "f32"),
    ("attention", "M=2,N=3,D=1,L=1", "128x128", "", "bf16"),
    ("layernorm-matmul", "M=3,N=3,K=2", "128x128", "M=64", "bf16"),
    ("rms-swiglu", "M=3,N=2,K=3,D=2", "128x128", "M=64", "bf16"),
]


@pytest.mark.gpu
@pytest.mark.parametrize("example,dims,block,lens,precision", VERIFY)
def test_verify_every_snapshot_against_reference_interpreter(example, dims, block, lens, precision):
    _, count = EXAMPLES[example]
    for k in range(1, count + 1):
        args = ["verify", PROGRAMS / example / f"snapshot_{k}.json", "--dims", dims, "--block", block,
                "--precision", precision, "--trials", 2]
        if lens:
            args += ["--len", lens]
        r = cli(*args, check=0)
        assert "verdict: equivalent" in r.stdout


# the block-program compiler route, float64 (host/bfgpu_codegen.cpp), on programs no fused kernel covers
GENERIC = [
    ("attention", "M=2,N=2,D=2,L=2", "4x4", ""),
    ("layernorm-matmul", "M=2,N=2,K=2", "4x4", ""),
    ("rms-swiglu", "M=2,N=2,K=2,D=2", "4x4", ""),
    ("rms-swiglu", "M=3,N=2,K=4,D=1", "4x4", "M=2,N=3,K=2,D=4"),  # asymmetric, test_engine.cpp:221-238
    ("attention", "M=3,N=2,D=1,L=2", "4x4", "M=2,N=3,D=4,L=2"),
]


@pytest.mark.gpu
@pytest.mark.parametrize("example,dims,block,lens", GENERIC)
def test_generic_route_runs_unfused_and_every_snapshot(example, dims, block, lens):
    _, count = EXAMPLES[example]
    files = ["lowered.json"] + [f"snapshot_{k}.json" for k in range(1, count + 1)]
    for f in files:
        args = ["verify", PROGRAMS / example / f, "--dims", dims, "--block", block, "--trials", 2, "--route", "generic"]
        if lens:
            args += ["--len", lens]
        r = cli(*args, check=0)
        assert "route: generic f64" in r.stdout and "verdict: equivalent" in r.stdout, f
    # auto routes the unfused program to the generic executor, the fused ones to their kernels
    r = cli("verify", PROGRAMS / example / "lowered.json", "--dims", dims, "--block", block, "--trials", 1,
            *(["--len", lens] if lens else []), check=0)
    assert "route: generic f64" in r.stdout
    r = cli("verify", PROGRAMS / example / "lowered.json", "--dims", dims, "--block", block, "--route", "fused", check=1)
    assert "no CPU fallback" in r.stderr


# The driver's peeling route (rule R7, `fuse --enable-peel`, off by default: engine.hpp:22,
# tools/blockfuse_main.cpp:122-126). Its final rms-swiglu snapshot splits the K map into a
# First map and a Rest map; with K bound to a single block the Rest range is empty and the
# reference zero-fills its accumulators from a probe iteration (interpreter.hpp:350-360),
# the case tests/acceptance.cpp:590-594 checks ("peeling stays sound when the remainder is empty").
PEEL = PROGRAMS / "rms-swiglu-peel"


def test_peel_route_files_regenerate_identically(tmp_path):
    cli("snapshots", "rms-swiglu", "--out-dir", tmp_path, "--enable-peel", check=0)
    for f in sorted(PEEL.glob("*.json")):
        assert (tmp_path / f.name).read_text() == f.read_text(), f.name
    final = json.loads((PEEL / "snapshot_2.json").read_text())

    def ranges(g):
        for n in g["nodes"]:
            if n.get("range"):
                yield n["dim"], n["range"]
            if n.get("inner"):
                yield from ranges(n["inner"])

    assert {("K", "first"), ("K", "rest")} <= set(ranges(final["graph"]))
    # the first snapshot is the default route's first snapshot (recognized, H buffered); the
    # peeled final snapshot is no fused kernel's canonical form, so it goes to the compiler
    assert (PEEL / "snapshot_1.json").read_text() == (PROGRAMS / "rms-swiglu" / "snapshot_1.json").read_text()
    assert "no CPU fallback" in cli("recognize", PEEL / "snapshot_2.json", check=1).stderr


PEEL_BINDINGS = [
    ("M=2,N=2,K=2,D=2", "4x4", ""),               # acceptance binding (tests/acceptance.cpp:175-201)
    ("M=3,N=2,K=4,D=1", "4x4", "M=2,N=3,K=2,D=4"),  # asymmetric (tests/test_engine.cpp:221-238)
    ("M=2,N=2,K=1,D=2", "4x4", "K=3"),             # singleton K: the Rest map is empty
    ("M=2,N=3,K=1,D=3", "4x4", "M=5,N=3,K=7,D=2"),  # empty Rest, ragged block lengths
]


@pytest.mark.gpu
@pytest.mark.parametrize("dims,block,lens", PEEL_BINDINGS)
def test_peel_route_on_the_compiler(dims, block, lens):
    for f in ("snapshot_1.json", "snapshot_2.json"):
        args = ["verify", PEEL / f, "--dims", dims, "--block", block, "--trials", 2, "--route", "generic"]
        if lens:
            args += ["--len", lens]
        r = cli(*args, check=0)
        assert "route: generic f64" in r.stdout and "verdict: equivalent" in r.stdout, (f, r.stdout)
    # auto: the unrecognized peeled snapshot runs on the compiler, never on the CPU
    r = cli("verify", PEEL / "snapshot_2.json", "--dims", dims, "--block", block, "--trials", 1,
            *(["--len", lens] if lens else []), check=0)
    assert "route: generic f64" in r.stdout and "verdict: equivalent" in r.stdout


@pytest.mark.gpu
def test_run_reports_output():
    r = cli("run", PROGRAMS / "rms-swiglu" / "snapshot_3.json", "--dims", "M=2,N=2,K=3,D=2", "--block", "128x128",
            "--repeat", 2, check=0)
    got = json.loads(r.stdout)
    assert got["output"] == "O" and got["rows"] == 256 and got["cols"] == 256
    assert got["rms"] > 0 and got["ms"] > 0
