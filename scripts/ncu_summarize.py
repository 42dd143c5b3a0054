"""Summarize ncu captures (.ncu-rep) into profiles/: key metrics per kernel launch.

    python scripts/ncu_summarize.py <tag> <rep> [<rep> ...]
Writes profiles/<tag>_<rep-stem>.txt and merges per-kernel numbers into profiles/ncu_summary.json
(the file bench.py reads for roofline.traffic).
"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor_active_pct_elapsed"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor_active_pct_active"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_throughput_pct"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_throughput_pct"),
    ("lts__t_sector_hit_rate.pct", "l2_hit_rate_pct"),
    ("sm__cycles_elapsed.avg.per_second", "sm_clock"),
    ("launch__registers_per_thread", "registers"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__inst_executed_pipe_uniform.sum", "uniform_inst"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem_wavefronts"),
    ("launch__shared_mem_per_block_dynamic", "dyn_smem"),
]
SCALE = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1, "ms": 1e-3, "us": 1e-6, "ns": 1e-9, "msecond": 1e-3,
         "usecond": 1e-6, "nsecond": 1e-9, "Ghz": 1e9, "Mhz": 1e6, "hz": 1}


def read(rep):
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")].split("(")[0]}
        for key, short in KEYS:
            if key in hdr:
                i = hdr.index(key)
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                d[short] = v * SCALE.get(units[i], 1) if units[i] in SCALE else v
                d[short + "_unit"] = units[i] if units[i] not in SCALE else ("s" if "s" in units[i] else ("Hz" if "hz" in units[i].lower() else "B"))
        res.append(d)
    return res


def main():
    tag, reps = sys.argv[1], sys.argv[2:]
    summ_path = ROOT / "profiles" / "ncu_summary.json"
    summ = json.loads(summ_path.read_text()) if summ_path.exists() else {}
    for rep in reps:
        rep = Path(rep)
        launches = read(rep)
        lines = [f"# ncu --set full --clock-control none capture: {rep.name} ({tag})"]
        for i, d in enumerate(launches):
            lines.append(f"\n## launch {i}: {d['kernel']}")
            for key, short in KEYS:
                if short in d:
                    lines.append(f"{key:70s} {d[short]:.6g} {d.get(short + '_unit', '')}")
            if "dram_read" in d:
                lines.append(f"{'dram bytes (read+write)':70s} {d['dram_read'] + d['dram_write']:.6g} B")
        (ROOT / "profiles" / f"{tag}_{rep.stem}.txt").write_text("\n".join(lines) + "\n")
        print("\n".join(lines))
        for d in launches:
            short = d["kernel"].split("::")[-1]
            entry = summ.setdefault(f"{short}@{rep.stem}", {})
            entry.update({"dram_bytes_per_launch": d.get("dram_read", 0) + d.get("dram_write", 0),
                          "duration_s": d.get("duration"), "tensor_active_pct_elapsed": d.get("tensor_active_pct_elapsed"),
                          "sm_clock_hz": d.get("sm_clock"), "source": f"profiles/{tag}_{rep.stem}.txt"})
    summ_path.write_text(json.dumps(summ, indent=1, sort_keys=True) + "\n")


if __name__ == "__main__":
    main()
