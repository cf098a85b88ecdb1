"""Summarise `ncu --set full` reports (one launch per kernel; several reports
comma-separated) into a
markdown table and profiles/traffic.json (DRAM bytes per launch, read by
bench.py for roofline.traffic).

  python tools/ncu_summary.py gpurun_out/r01b_step_full.ncu-rep r01 "command line"
"""
import csv
import io
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % peak"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %"),
    ("launch__registers_per_thread", "regs"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("smsp__inst_executed.sum", "warp inst"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) pipe %"),
    ("smsp__cycles_elapsed.avg.per_second", "SM clock"),
]
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
         "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0,
         "msecond": 1e-3, "second": 1.0, "cycle/nsecond": 1e9, "cycle/usecond": 1e6,
         "cycle/msecond": 1e3, "cycle/second": 1.0, "Ghz": 1e9, "Mhz": 1e6, "hz": 1.0}


def short(name: str) -> str:
    name = re.sub(r"\(.*", "", name)
    name = re.sub(r"^.*::", "", name)
    return name.replace("void ", "")


def main(reps: str, tag: str, command: str):
    seen, table, traffic = {}, [], {}
    for rep in reps.split(","):
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                             text=True, check=True).stdout
        rows = list(csv.reader(io.StringIO(raw)))
        summarise(rows, seen, table, traffic, tag)
    write(tag, command, table, traffic)


def summarise(rows, seen, table, traffic, tag):
    hdr, units = rows[0], rows[1]
    ki = hdr.index("Kernel Name")
    for r in rows[2:]:
        k = short(r[ki])
        seen[k] = seen.get(k, 0) + 1
        if seen[k] > 1:
            continue
        vals = {}
        for m, _ in METRICS:
            if m not in hdr:
                vals[m] = float("nan")
                continue
            i = hdr.index(m)
            v = float(r[i].replace(",", "")) if r[i] not in ("", "n/a") else float("nan")
            vals[m] = v * SCALE.get(units[i], 1.0) if units[i] in SCALE else v
        table.append((k, vals))
        traffic[k] = {"dram_bytes_per_launch": vals["dram__bytes_read.sum"] + vals["dram__bytes_write.sum"],
                      "issue_active_pct": vals["smsp__issue_active.avg.pct_of_peak_sustained_active"],
                      "warp_inst_per_launch": vals["smsp__inst_executed.sum"],
                      "fma_pipe_pct": vals["sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"],
                      "xu_pipe_pct": vals["sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"],
                      "ncu_time_s": vals["gpu__time_duration.sum"],
                      "ncu_sm_hz": vals["smsp__cycles_elapsed.avg.per_second"],
                      "source": f"profiles/{tag}_ncu_step.md"}


def write(tag, command, table, traffic):
    lines = [f"# {tag}: ncu --set full, one launch per step kernel", "",
             f"Command: `{command}`", "",
             "Cold-cache, serialised replay with clocks unlocked (`--clock-control none`): compare "
             "shares and ratios, not absolute times (bench.py times the same kernels with CUDA events).",
             "", "| kernel | " + " | ".join(lbl for _, lbl in METRICS) + " |",
             "|---" * (len(METRICS) + 1) + "|"]
    for k, v in table:
        cells = []
        for m, _ in METRICS:
            x = v[m]
            if m == "gpu__time_duration.sum":
                cells.append(f"{x * 1e6:.1f} us")
            elif m.startswith("dram__bytes"):
                cells.append(f"{x / 1e6:.1f} MB")
            elif m == "smsp__inst_executed.sum":
                cells.append(f"{x / 1e6:.1f} M")
            elif m == "smsp__cycles_elapsed.avg.per_second":
                cells.append(f"{x / 1e6:.0f} MHz")
            else:
                cells.append(f"{x:.1f}")
        lines.append(f"| {k} | " + " | ".join(cells) + " |")
    out_md = os.path.join(ROOT, "profiles", f"{tag}_ncu_step.md")
    with open(out_md, "w") as f:
        f.write("\n".join(lines) + "\n")
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    old = {}
    if os.path.exists(tp):
        with open(tp) as f:
            old = json.load(f)
    old.update(traffic)
    with open(tp, "w") as f:
        json.dump(old, f, indent=1, sort_keys=True)
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "")
