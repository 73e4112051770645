"""Summarise an ncu report (--set full) or an ncu launch-list CSV into a small text file.

python tools/ncu_summary.py full REPORT.ncu-rep CONFIGS_PER_LAUNCH > out.txt
python tools/ncu_summary.py launches LAUNCHES.csv > out.txt
"""
import csv
import io
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "launch__occupancy_limit_registers", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum", "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum",
    "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "sm__cycles_elapsed.avg.per_second",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
]


def full(path, configs):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        print(f"kernel: {d.get('Kernel Name')}")
        for m in METRICS:
            if m in d:
                print(f"  {m:80s} {d[m]:>20s} {u.get(m, '')}")
        try:
            inst = float(d["smsp__inst_executed.sum"].replace(",", ""))
            fp = sum(float(d[m].replace(",", "")) for m in METRICS if m.startswith("smsp__sass_thread_inst_executed_op_d"))
            print(f"  warp instructions per configuration: {inst * 32 / configs:.2f} (thread-level)")
            print(f"  FP64 thread instructions per configuration (dadd+dmul+dfma): {fp / configs:.2f}")
        except Exception:
            pass


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = {}
    order = []
    for r in rows:
        if len(r) > 5 and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d["Metric Name"] != "gpu__time_duration.sum":
                continue
            name = d["Kernel Name"].split("(")[0]
            if name not in agg:
                agg[name] = [0, 0.0]
                order.append(name)
            agg[name][0] += 1
            agg[name][1] += float(d["Metric Value"].replace(",", ""))
    tot = sum(v[1] for v in agg.values())
    print(f"{'kernel':60s} {'launches':>8s} {'total us':>12s} {'share':>7s}")
    for n in order:
        c, t = agg[n]
        print(f"{n[:60]:60s} {c:8d} {t / 1e3:12.1f} {t / tot:7.3f}")


if __name__ == "__main__":
    if sys.argv[1] == "full":
        full(sys.argv[2], float(sys.argv[3]))
    else:
        launches(sys.argv[2])
