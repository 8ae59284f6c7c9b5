"""Pipe / traffic counters per kernel from an ncu --set full report (raw page).

    python tools/ncu_raw.py report.ncu-rep [kernel-substring] > summary.txt

Prints, per captured launch: duration, FP64 pipe activity (DFMA/DADD/DMUL and
DMMA share one FP64 pipe on sm_100), the FP64 tensor-path ops, executed FP64
thread instructions, DRAM bytes read/written, occupancy and issue activity.
"""
import csv
import io
import re
import subprocess
import sys

WANT = [
    r"^gpu__time_duration\.sum$",
    r"^sm__pipe_fp64_cycles_active\.avg\.pct_of_peak_sustained_(active|elapsed)$",
    r"^sm__inst_executed_pipe_fp64\.avg\.pct_of_peak_sustained_active$",
    r"^sm__ops_path_tensor_src_fp64\.(sum|avg\.pct_of_peak_sustained_(active|elapsed))$",
    r"^sm__pipe_tensor_op_dmma_cycles_active\.avg\.pct_of_peak_sustained_(active|elapsed)$",
    r"^sm__inst_executed_pipe_fp64.*\.sum$",
    r"^smsp__sass_thread_inst_executed_op_d(add|mul|fma)_pred_on\.sum$",
    r"^smsp__sass_thread_inst_executed\.sum$",
    r"^smsp__inst_executed\.sum$",
    r"^dram__bytes_(read|write)\.sum$",
    r"^sm__warps_active\.avg\.pct_of_peak_sustained_active$",
    r"^sm__inst_issued\.avg\.pct_of_peak_sustained_active$",
    r"^launch__registers_per_thread$",
    r"^launch__grid_size$",
    r"^launch__block_size$",
    r"^sm__throughput\.avg\.pct_of_peak_sustained_elapsed$",
    r"^gpu__compute_memory_throughput\.avg\.pct_of_peak_sustained_elapsed$",
]


def main():
    rep = sys.argv[1]
    kf = sys.argv[2] if len(sys.argv) > 2 else None
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    if len(rows) < 3:
        print("no data")
        return
    head, units = rows[0], rows[1]
    cols = [i for i, n in enumerate(head) if any(re.match(w, n) for w in WANT)]
    kcol = head.index("Kernel Name")
    for r in rows[2:]:
        if kf and kf not in r[kcol]:
            continue
        print(r[kcol][:100])
        for i in cols:
            if i < len(r) and r[i] not in ("", "n/a"):
                print(f"    {head[i]:70s} {r[i]:>18s} {units[i]}")


if __name__ == "__main__":
    main()
