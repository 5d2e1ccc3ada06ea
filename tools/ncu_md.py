"""Per-kernel ncu summary table from exported raw pages.

    python tools/ncu_md.py <dir> <tag> <key:label,...> > profiles/<tag>_ncu_....md

Reads <dir>/raw_<tag>_<key>.csv (`ncu -i rep --page raw --csv`, one kernel each) and
prints a markdown table of the metrics the design discussion uses, the real DRAM
bandwidth per kernel and the sum of the DRAM traffic.
"""
import csv
import sys

M = [("gpu__time_duration.sum", "time"), ("dram__bytes_read.sum", "DRAM read"), ("dram__bytes_write.sum", "DRAM write"),
     ("lts__t_sector_hit_rate.pct", "L2 hit %"), ("l1tex__t_sector_hit_rate.pct", "L1 hit %"),
     ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
     ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
     ("smsp__thread_inst_executed_per_inst_executed.ratio", "threads / inst"),
     ("launch__registers_per_thread", "registers"), ("smsp__inst_executed.sum", "warp instructions"),
     ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "shared wavefronts % peak"),
     ("l1tex__data_pipe_lsu_wavefronts.sum.pct_of_peak_sustained_elapsed", "L1TEX LSU wavefronts % peak"),
     ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe %"),
     ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %")]
ST = ["long_scoreboard", "barrier", "wait", "short_scoreboard", "math_pipe_throttle", "not_selected", "lg_throttle",
      "mio_throttle", "branch_resolving", "dispatch_stall", "no_instruction"]
BY = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
TM = {"ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1}

d_, tag, spec = sys.argv[1], sys.argv[2], sys.argv[3]
K = [tuple(x.split(":", 1)) for x in spec.split(",")]
D = {}
for k, _ in K:
    rows = list(csv.reader(open(f"{d_}/raw_{tag}_{k}.csv")))
    hdr, units, r = rows[0], rows[1], rows[2]
    D[k] = {h: (r[i], units[i]) for i, h in enumerate(hdr)}


def val(k, m):
    v, u = D[k].get(m, ("n/a", ""))
    try:
        f = float(v)
        v = f"{f:.4g}" if abs(f) < 1e6 else f"{f:.4e}"
    except ValueError:
        pass
    return f"{v} {u}".strip()


print("| metric | " + " | ".join(n for _, n in K) + " |")
print("|---|" + "---|" * len(K))
print("| kernel | " + " | ".join(D[k].get("Kernel Name", ("", ""))[0][:60] for k, _ in K) + " |")
for m, n in M:
    print(f"| {n} | " + " | ".join(val(k, m) for k, _ in K) + " |")
for s in ST:
    m = f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio"
    print(f"| stall {s} (per issue) | " + " | ".join(val(k, m) for k, _ in K) + " |")
print()
tot = 0.0
for k, n in K:
    b = sum(float(D[k][m][0]) * BY[D[k][m][1]] for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
    t = float(D[k]["gpu__time_duration.sum"][0]) * TM[D[k]["gpu__time_duration.sum"][1]]
    tot += b
    print(f"* {n}: {b / 1e9:.1f} GB of DRAM traffic in {t * 1e3:.1f} ms = {b / t / 1e12:.2f} TB/s")
print(f"\nSum of the DRAM traffic of these kernels: {tot / 1e9:.1f} GB")
