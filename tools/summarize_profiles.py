"""Summarise a round's ncu captures into profiles/ (tracked).

    python tools/summarize_profiles.py <tag> [config]

Reads gpurun_out/launches_<tag>.csv (per-launch device times, one bench step
+ warmup + e2e steps) and gpurun_out/prof_<tag>_<kernel>.ncu-rep (one
`--set full` capture per listing kernel) and writes
  profiles/<tag>_launches_<config>.csv   (copy of the launch list)
  profiles/<tag>_ncu_<config>.md         (key metrics per kernel)
  profiles/traffic.json                  (DRAM bytes per listing step, read by bench.py)
"""
import csv
import io
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")
KERNELS = ["reg", "warp", "cta_c1", "cta_c2"]
METRICS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % peak"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("l1tex__data_pipe_lsu_wavefronts.sum.pct_of_peak_sustained_elapsed", "L1TEX LSU wavefronts % peak"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "shared wavefronts % peak"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "threads / inst"),
    ("launch__registers_per_thread", "registers"),
    ("launch__occupancy_limit_registers", "CTAs/SM by regs"),
    ("launch__occupancy_limit_shared_mem", "CTAs/SM by smem"),
]
STALLS = ["long_scoreboard", "short_scoreboard", "wait", "barrier", "not_selected", "math_pipe_throttle",
          "lg_throttle", "mio_throttle", "branch_resolving"]


def raw(rep):
    exported = rep.replace("/prof_", "/raw_").replace(".ncu-rep", ".csv")
    if os.path.exists(exported):
        txt = open(exported).read()
    else:
        txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    if len(rows) < 3:
        return None
    hdr, units, r = rows[0], rows[1], rows[2]
    return {h: (r[i], units[i]) for i, h in enumerate(hdr)}


def to_bytes(v, u):
    f = float(v)
    return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(u, 1)


def main():
    tag = sys.argv[1]
    cfg = sys.argv[2] if len(sys.argv) > 2 else "c4"
    os.makedirs(PROF, exist_ok=True)
    lsrc = os.path.join(OUT, f"launches_{tag}.csv")
    if os.path.exists(lsrc):
        shutil.copy(lsrc, os.path.join(PROF, f"{tag}_launches_{cfg}.csv"))
    lines = [f"# ncu summary `{tag}` ({cfg}, degree ordering, A+-, count+checksum)", "",
             "One `ncu --set full --clock-control none` capture per listing kernel "
             "(tools/profile_all.sh); cold-cache, serialised replays.", ""]
    lines.append("| metric | " + " | ".join(KERNELS) + " |")
    lines.append("|---|" + "---|" * len(KERNELS))
    data = {k: raw(os.path.join(OUT, f"prof_{tag}_{k}.ncu-rep")) for k in KERNELS}
    for m, label in METRICS:
        cells = []
        for k in KERNELS:
            d = data[k]
            cells.append(f"{d[m][0]} {d[m][1]}".strip() if d and m in d else "n/a")
        lines.append(f"| {label} | " + " | ".join(cells) + " |")
    for st in STALLS:
        key = f"smsp__average_warps_issue_stalled_{st}_per_issue_active.ratio"
        cells = [data[k][key][0] if data[k] and key in data[k] else "n/a" for k in KERNELS]
        lines.append(f"| stall {st} (per issue) | " + " | ".join(cells) + " |")
    total = 0.0
    ok = True
    for k in KERNELS:
        d = data[k]
        if not d or "dram__bytes_read.sum" not in d:
            ok = False
            continue
        total += to_bytes(*d["dram__bytes_read.sum"]) + to_bytes(*d["dram__bytes_write.sum"])
    lines += ["", f"DRAM traffic of one listing step (sum over the class kernels): "
              f"{total / 1e9:.1f} GB" + ("" if ok else " (incomplete: some captures missing)")]
    with open(os.path.join(PROF, f"{tag}_ncu_{cfg}.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    tp = os.path.join(PROF, "traffic.json")
    tj = json.load(open(tp)) if os.path.exists(tp) else {}
    if ok:
        tj[f"{cfg}:degree:apm"] = total
    with open(tp, "w") as f:
        json.dump(tj, f, indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
