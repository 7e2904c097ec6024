"""Summarise an .ncu-rep: key throughput metrics + top stall reasons (run here, no GPU)."""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.per_cycle_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread",
        "smsp__inst_executed.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed"]


def main(path, kernel_filter=None):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units = rows[0], rows[1]
    for row in rows[2:]:
        d = dict(zip(head, row))
        name = d.get("Kernel Name", "")
        if kernel_filter and kernel_filter not in name:
            continue
        print("kernel:", name[:100])
        for k in KEYS:
            if k in d:
                print(f"  {k:70s} {d[k]} {units[head.index(k)]}")
        stalls = []
        for k, v in d.items():
            if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued"):
                try:
                    stalls.append((float(v.replace(",", "")), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        tot = sum(s for s, _ in stalls) or 1.0
        print("  stall samples:", ", ".join(f"{n} {100 * s / tot:.0f}%" for s, n in sorted(stalls, reverse=True)[:8]))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
