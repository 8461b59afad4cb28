"""Summarise ncu captures into profiles/ (markdown + per-workload DRAM traffic).

    python tools/ncu_summary.py TAG workload=path.ncu-rep [workload=path.ncu-rep ...]

Writes profiles/<TAG>_ncu_summary.md and merges {workload: bytes per launch}
into profiles/ncu_traffic.json (bench.py reads it for roofline.traffic).
"""

import csv
import io
import json
import subprocess
import sys
from pathlib import Path

REPO = Path(__file__).resolve().parents[1]
KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of peak"),
    ("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", "DMMA pipe %"),
    ("sm__inst_executed_pipe_fp64_op_dmma.sum", "DMMA instructions"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def raw(path: str) -> list[dict]:
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {}
        for h, u, v in zip(hdr, units, r):
            d[h] = (v, u)
        res.append(d)
    return res


def to_bytes(v: str, u: str) -> float:
    return float(v.replace(",", "")) * SCALE.get(u, 1)


def main() -> None:
    tag = sys.argv[1]
    md = [f"# ncu summary ({tag})", "",
          "`ncu --set full --clock-control none --import-source on`, one launch per capture "
          "(replayed; cold-cache, serialised — compare shares, not absolutes).", ""]
    traffic_path = REPO / "profiles" / "ncu_traffic.json"
    traffic = json.loads(traffic_path.read_text()) if traffic_path.exists() else {}
    for arg in sys.argv[2:]:
        wl, path = arg.split("=", 1)
        for d in raw(path):
            name = d.get("Kernel Name", ("?", ""))[0]
            md += [f"## {wl}: `{name[:110]}`", "", "| metric | value | unit |", "|---|---|---|"]
            for k, label in KEYS:
                if k in d:
                    v, u = d[k]
                    md.append(f"| {label} (`{k}`) | {v} | {u} |")
            if "dram__bytes_read.sum" in d and "dram__bytes_write.sum" in d:
                tb = to_bytes(*d["dram__bytes_read.sum"]) + to_bytes(*d["dram__bytes_write.sum"])
                traffic[wl] = int(tb)
                md.append(f"| DRAM read+write per launch | {int(tb)} | byte |")
            md.append("")
    (REPO / "profiles" / f"{tag}_ncu_summary.md").write_text("\n".join(md) + "\n")
    traffic_path.write_text(json.dumps(traffic, indent=1) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    main()
