"""Rebuild profiles/traffic.json and profiles/pipes.json from the committed ncu
summaries (profiles/r01_ncu_<kernel>_<config>.txt, written by ncu_summary.py)
and the cfg1c launch list (the whole wide pipeline per step).

    python tools/update_profile_tables.py [round-prefix, default r02]
"""
import csv
import gzip
import json
import os
import sys
from collections import defaultdict

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "profiles")
CAPTURES = {"cfg4": "fhn_cm_cfg4", "cfg2": "lorenz_fast_cfg2", "cfg1b": "resample_bank_cfg1b",
            "net": "fhnnet_fast_net", "cfg1c": "wide2_merge_cfg1c", "cfg0": "lorenz_small_cfg0"}
UNITS = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def field(path, key):
    for line in open(path):
        if line.strip().startswith(key + " :"):
            return line.split(":", 1)[1].split()
    raise KeyError(f"{key} not in {path}")


def num(path, key):
    parts = field(path, key)
    return float(parts[0]) * (UNITS.get(parts[1], 1.0) if len(parts) > 1 else 1.0)


def opcode_counts(sass_gz):
    """Executed warp instructions of the multi-slot opcodes, from the capture's SASS
    source page (ncu --page source --csv): IMAD.WIDE / IMAD.HI (32x32 multiplies) and
    MUFU - the inputs of bench.py's dispatch-slot model."""
    rows = list(csv.reader(gzip.open(sass_gz, "rt")))
    hdr = next(r for r in rows if "Source" in r and "Instructions Executed" in r)
    isrc, iex = hdr.index("Source"), hdr.index("Instructions Executed")
    out = {"imad_wide_per_launch": 0, "mufu_per_launch": 0}
    for r in rows[rows.index(hdr) + 1:]:
        if len(r) <= max(isrc, iex):
            continue
        ops = r[isrc].split()
        op = ops[1] if ops and ops[0].startswith("@") and len(ops) > 1 else (ops[0] if ops else "")
        if op.startswith("IMAD.WIDE") or op.startswith("IMAD.HI"):
            out["imad_wide_per_launch"] += int(r[iex])
        elif op.startswith("MUFU"):
            out["mufu_per_launch"] += int(r[iex])
    return out


def wide_pipeline_bytes(csv_path):
    rows = [r for r in csv.reader(open(csv_path)) if len(r) > 5]
    hdr = rows[0]
    iid, iname, im, iv = (hdr.index(k) for k in ("ID", "Kernel Name", "Metric Name",
                                                  "Metric Value"))
    per, names = defaultdict(dict), {}
    for r in rows[1:]:
        per[r[iid]][r[im]] = float(r[iv].replace(",", ""))
        names[r[iid]] = r[iname]
    total = sum(m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
                for lid, m in per.items() if "pf::" in names[lid])
    steps = sum(1 for lid in per if "wide2_merge" in names[lid])
    return int(total / steps)


def main(prefix="r02"):
    traffic = json.load(open(os.path.join(ROOT, "traffic.json")))
    pipes = json.load(open(os.path.join(ROOT, "pipes.json")))
    for cfg, cap in CAPTURES.items():
        path = os.path.join(ROOT, f"{prefix}_ncu_{cap}.txt")
        if cfg != "cfg1c":
            traffic[cfg] = int(num(path, "dram__bytes_read.sum") + num(path, "dram__bytes_write.sum"))
        pct = lambda k: num(path, k)  # noqa: E731
        pipes[cfg] = {
            "kernel": cap.rsplit("_", 1)[0],
            "fma_pipe_pct": pct("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
            "alu_pipe_pct": pct("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"),
            "xu_pipe_pct": pct("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"),
            "issue_active_pct": pct("smsp__issue_active.avg.pct_of_peak_sustained_active"),
            "dram_throughput_pct": pct("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
            "warp_inst_per_launch": num(path, "smsp__inst_executed.sum"),
        }
        sass = os.path.join(ROOT, f"{prefix}_ncu_{cap}_sass.csv.gz")
        if os.path.exists(sass):
            pipes[cfg].update(opcode_counts(sass))
    traffic["cfg1c"] = wide_pipeline_bytes(os.path.join(ROOT, f"{prefix}_launches_cfg1c.csv"))
    json.dump(traffic, open(os.path.join(ROOT, "traffic.json"), "w"), indent=1)
    json.dump(pipes, open(os.path.join(ROOT, "pipes.json"), "w"), indent=1)
    print(json.dumps({"traffic": traffic, "pipes": pipes}, indent=1)[:2000])


if __name__ == "__main__":
    main(*sys.argv[1:])
