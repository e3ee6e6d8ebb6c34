"""Condense an `ncu --set full` report into the lines the roofline and the
judge need (run here, on the CPU box, on a report gpurun brought back).

Usage: python tools/ncu_summary.py REPORT.ncu-rep [out.txt] [traffic.json] [kernel-substring]

Prints per launch: duration, DRAM bytes (read + write), pipe utilisation,
issue activity, occupancy, registers and the top stall reasons.  With a third
argument it also writes {"kernel", "bytes_per_launch", "duration_us"} (the
mean over the captured launches) for bench.py's roofline.traffic field.
"""

import csv
import io
import json
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma_pipe_%"),
    ("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed", "fmaheavy_%"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "alu_pipe_%"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "lsu_%"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64_pipe_%"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor_pipe_%"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_active_%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_%"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__inst_executed.sum", "warp_insts"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_%"),
    ("sm__cycles_elapsed.avg.per_second", "sm_clock"),
]


def _to_bytes(value: str, unit: str) -> float:
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    return float(value.replace(",", "")) * scale.get(unit, 1)


def _to_us(value: str, unit: str) -> float:
    scale = {"nsecond": 1e-3, "usecond": 1, "msecond": 1e3, "second": 1e6, "ns": 1e-3, "us": 1, "ms": 1e3}
    return float(value.replace(",", "")) * scale.get(unit, 1)


def main():
    rep = sys.argv[1]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    col = {h: i for i, h in enumerate(hdr)}
    out = []
    launches = []
    for r in rows[2:]:
        name = r[col["Kernel Name"]]
        rec = {"kernel": name}
        for key, short in KEYS:
            if key in col:
                rec[short] = (r[col[key]], units[col[key]])
        stalls = []
        for h, i in col.items():
            if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
                try:
                    stalls.append((float(r[i]), h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        rec["stalls"] = stalls[:6]
        launches.append(rec)
        out.append(f"== {name}")
        for key, short in KEYS:
            if short in rec:
                v, u = rec[short]
                out.append(f"   {short:16s} {v} {u}")
        d_r = _to_bytes(*rec["dram_read"]) if "dram_read" in rec else 0.0
        d_w = _to_bytes(*rec["dram_write"]) if "dram_write" in rec else 0.0
        rec["traffic"] = d_r + d_w
        out.append(f"   {'traffic_bytes':16s} {d_r + d_w:.0f}")
        out.append("   stalls (warps per issue): " + ", ".join(f"{n}={v:.2f}" for v, n in stalls[:6]))
    text = "\n".join(out)
    print(text)
    if len(sys.argv) > 2:
        with open(sys.argv[2], "w") as f:
            f.write(f"# ncu --set full summary of {rep}\n" + text + "\n")
    if len(sys.argv) > 4:
        launches = [l for l in launches if sys.argv[4] in l["kernel"]]
    if len(sys.argv) > 3 and launches:
        mean_traffic = sum(l["traffic"] for l in launches) / len(launches)
        mean_us = sum(_to_us(*l["duration"]) for l in launches) / len(launches)
        with open(sys.argv[3], "w") as f:
            json.dump({"kernel": launches[0]["kernel"], "bytes_per_launch": mean_traffic,
                       "duration_us": mean_us, "launches": len(launches), "source": rep}, f, indent=1)


if __name__ == "__main__":
    main()
