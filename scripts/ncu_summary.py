"""Summarise an ncu report (--page raw) per kernel: duration, DRAM bytes, SOL %, FP64 pipe, occupancy, top stalls."""
import csv, subprocess, sys, io

def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "smsp__inst_executed.sum", "sm__instruction_throughput.avg.pct_of_peak_sustained_active",
        "lts__t_bytes.sum", "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "sm__inst_executed.avg.per_cycle_active"]

def main(rep):
    h, units, rows = raw(rep)
    idx = {k: i for i, k in enumerate(h)}
    pre, suf = "smsp__average_warps_issue_stalled_", "_per_issue_active.ratio"
    stall_cols = [k for k in h if k.startswith(pre) and k.endswith(suf)]
    for r in rows:
        name = r[idx["Kernel Name"]][:60]
        print("==", name)
        for k in KEYS:
            if k in idx:
                print(f"   {k:70s} {r[idx[k]]:>14s} {units[idx[k]]}")
        st = []
        for k in stall_cols:
            try:
                st.append((float(r[idx[k]]), k[len(pre):-len(suf)]))
            except ValueError:
                pass
        st.sort(reverse=True)
        print("   stalls:", ", ".join(f"{n}={v:.2f}" for v, n in st[:6]))

if __name__ == "__main__":
    main(sys.argv[1])
