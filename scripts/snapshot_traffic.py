"""Modeled vs measured global-memory bytes for every program the fusion driver produces
(SURVEY.md §8(f)3): the unfused lower() output and each fusion snapshot, on the GPU.

For each example, each program file (lowered.json, snapshot_k.json) runs once through the
drop-in (bfgpu-cli run -> bfgpu::execute) under ncu, and the DRAM bytes of its kernels are
summed and set beside the reference's own traffic_bytes model (metrics.hpp:154-191) at the
same binding (tests/golden/traffic_model.json, made from the reference compiled in place):

  route "generic"  every program file on the float64 block-program compiler: one generated
                   kernel per top-level operator, the reference's execution model (model with
                   element_bytes 8);
  route "kernels"  each snapshot on its bf16 tensor-core plan (element_bytes 2): the final
                   snapshots on the fused kernels, the first snapshots on the staged plans.

The adapter's layout transposes (bf_transpose: host column-major <-> device row-major) are
reported apart: the model counts a program's inputs and outputs once, in place.
ncu flushes the caches before every kernel, so each kernel's bytes are its compulsory traffic,
which is what the model charges.

    python scripts/snapshot_traffic.py            # on the GPU box; writes gpurun_out/snapshot_traffic.json
"""
from __future__ import annotations

import csv
import io
import json
import subprocess
import sys
import tempfile
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
CLI = ROOT / "paper_2505_07829_b200" / "lib" / "bfgpu-cli"
MODEL = json.loads((ROOT / "tests" / "golden" / "traffic_model.json").read_text())["runs"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "ms": 1e-3,
         "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3}


def ncu_run(args: list[str]) -> dict:
    with tempfile.TemporaryDirectory() as d:
        log = Path(d) / "ncu.csv"
        cmd = ["ncu", "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum", "--csv",
               "--log-file", str(log), str(CLI)] + args
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=1800)
        if r.returncode != 0:
            return {"error": (r.stderr or r.stdout)[-500:]}
        lines = log.read_text().splitlines()
        start = [i for i, l in enumerate(lines) if l.startswith('"ID"')][0]
        rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
    h = rows[0]
    ik, im, iu, iv, iid = (h.index(k) for k in ("Kernel Name", "Metric Name", "Metric Unit", "Metric Value", "ID"))
    prog = {"bytes": 0.0, "time_s": 0.0, "launches": set(), "names": set()}
    layout = {"bytes": 0.0, "launches": set()}
    for r in rows[1:]:
        v = float(r[iv].replace(",", "")) * SCALE.get(r[iu], 1)
        tgt = layout if "transpose" in r[ik] else prog
        tgt["launches"].add(r[iid])
        if tgt is prog:
            prog["names"].add(r[ik].split("(")[0])
        if r[im].startswith("dram__bytes"):
            tgt["bytes"] += v
        elif r[im] == "gpu__time_duration.sum" and tgt is prog:
            prog["time_s"] += v
    return {"dram_bytes": prog["bytes"], "kernel_launches": len(prog["launches"]),
            "serialized_kernel_time_s": prog["time_s"], "kernels": sorted(prog["names"])[:8],
            "layout_transpose_bytes": layout["bytes"], "layout_launches": len(layout["launches"])}


def main() -> None:
    out = {"method": __doc__.split("\n\n")[0], "rows": []}
    for ex, ent in MODEL.items():
        with tempfile.TemporaryDirectory() as d:
            subprocess.run([str(CLI), "snapshots", ex, "--out-dir", d], check=True, capture_output=True)
            files = ["lowered"] + sorted(k for k in ent["model_bytes"]["generic"] if k.startswith("snapshot_"))
            for name in files:
                path = Path(d) / f"{name}.json"  # `snapshots` also writes the reference's lower() output
                for route in ("generic", "kernels"):
                    if route == "kernels" and name == "lowered":
                        continue
                    dims, lens = ent["spec"][route].split(" --len ")
                    args = ["run", str(path), "--dims", dims, "--block", "128x128", "--len", lens, "--route",
                            "generic" if route == "generic" else "fused", "--precision", "bf16", "--repeat", "1"]
                    m = ncu_run(args)
                    model = ent["model_bytes"][route][name]
                    row = {"example": ex, "program": name, "route": route, "binding": ent["spec"][route],
                           "model_bytes": model, "internal_buffered_edges": ent["internal_buffered_edges"][name],
                           "model_kernels": ent["kernels"][name], **m}
                    if "dram_bytes" in m:
                        row["measured_over_model"] = m["dram_bytes"] / model
                    out["rows"].append(row)
                    print(json.dumps(row), flush=True)
    dst = ROOT / "gpurun_out" / "snapshot_traffic.json"
    dst.parent.mkdir(exist_ok=True)
    dst.write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    sys.exit(main())
