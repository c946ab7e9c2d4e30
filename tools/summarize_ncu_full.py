"""Key metrics of one `ncu --set full` capture (one kernel launch) for profiles/.

    python tools/summarize_ncu_full.py gpurun_out/r1_kd_a0.ncu-rep > profiles/r1_kd_tc_alpha0_ncu.txt
"""
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "lts__t_bytes.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic", "launch__grid_size", "launch__block_size",
]


def main(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, u, v = rows[0], rows[1], rows[2]
    name = v[h.index("Kernel Name")]
    print(f"# {rep}\n# kernel: {name}")
    for k in KEYS:
        for i, c in enumerate(h):
            if c == k:
                print(f"{k:80s} {v[i]:>20s} {u[i]}")
    print("# warp stall samples (smsp__pcsamp_warps_issue_stalled_*)")
    st = []
    for i, c in enumerate(h):
        if c.startswith("smsp__pcsamp_warps_issue_stalled_") and not c.endswith("not_issued"):
            try:
                st.append((float(v[i].replace(",", "")), c[len("smsp__pcsamp_warps_issue_stalled_"):]))
            except ValueError:
                pass
    tot = sum(x for x, _ in st) or 1.0
    for x, c in sorted(st, reverse=True):
        if x > 0:
            print(f"  {c:30s} {x:12.0f} {100 * x / tot:6.2f}%")


if __name__ == "__main__":
    main(sys.argv[1])
