"""Summarise ncu evidence into small committed files (run in the build container).

    python profiles/summarize.py rep  <name> <file.ncu-rep>     -> profiles/<name>.json
    python profiles/summarize.py list <name> <launches.csv>     -> profiles/<name>.json

`rep` keeps the metrics the DESIGN/roofline discussion cites (duration, DRAM
bytes, pipe utilisation, occupancy, stall reasons); `list` aggregates an
`ncu --metrics gpu__time_duration.sum` launch list per kernel (share of time).
"""

from __future__ import annotations

import csv
import io
import json
import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent

KEEP = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_static",
    "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "sm__cycles_elapsed.avg.per_second",
    "lts__t_sectors_op_red.sum", "lts__t_requests_op_red.sum", "lts__t_sectors_op_atom.sum",
    "l1tex__t_requests_pipe_lsu_mem_global_op_red.sum", "lts__t_sectors_op_red_lookup_hit.sum",
]


def _raw(rep: Path):
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [dict(zip(hdr, r)) for r in rows[2:]], dict(zip(hdr, units))


def summarize_rep(name: str, rep: Path):
    recs, units = _raw(rep)
    res = []
    for d in recs:
        item = {"kernel": d.get("Kernel Name", "")[:120]}
        for k in KEEP:
            if k in d:
                item[k] = f"{d[k]} {units.get(k, '')}".strip()
        stalls = {}
        for k, v in d.items():
            if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
                try:
                    if float(v) >= 0.1:
                        stalls[k.split("stalled_")[1].split("_per_issue")[0]] = float(v)
                except ValueError:
                    pass
        item["stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1]))
        res.append(item)
    out = HERE / f"{name}.json"
    out.write_text(json.dumps({"source": rep.name, "kernels": res}, indent=1))
    print(out)


def summarize_list(name: str, path: Path):
    text = path.read_text().splitlines()
    start = next(i for i, l in enumerate(text) if l.startswith('"ID"'))
    rows = list(csv.DictReader(io.StringIO("\n".join(text[start:]))))
    agg = {}
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        k = r["Kernel Name"].split("(")[0][:90]
        unit = r.get("Metric Unit", "")
        v = float(r["Metric Value"].replace(",", ""))
        v_us = v / 1000.0 if unit in ("nsecond", "ns") else (v if unit in ("usecond", "us") else v * 1e3)
        a = agg.setdefault(k, {"launches": 0, "total_us": 0.0})
        a["launches"] += 1
        a["total_us"] += v_us
    tot = sum(a["total_us"] for a in agg.values()) or 1.0
    for a in agg.values():
        a["avg_us"] = a["total_us"] / a["launches"]
        a["share"] = a["total_us"] / tot
    out = HERE / f"{name}.json"
    out.write_text(json.dumps({"source": path.name, "note": "ncu --clock-control none, serialised "
                               "cold-cache launches: compare shares, not absolutes",
                               "kernels": dict(sorted(agg.items(), key=lambda kv: -kv[1]["total_us"]))},
                              indent=1))
    print(out)


if __name__ == "__main__":
    mode, name, path = sys.argv[1], sys.argv[2], Path(sys.argv[3])
    (summarize_rep if mode == "rep" else summarize_list)(name, path)
