"""Summarise an `ncu --set full` report: per kernel launch the headline
throughputs, occupancy, registers, DRAM bytes and the top warp-stall reasons.

    python tools/ncu_full_summary.py gpurun_out/<rep>.ncu-rep > profiles/<round>_full_summary.txt
"""
import csv
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration_ns"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_%"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "mem_%"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "l1_%"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "l2_%"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram_%"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_%"),
    ("launch__registers_per_thread", "regs"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_%"),
    ("l1tex__t_sector_hit_rate.pct", "l1_hit_%"),
    ("lts__t_sector_hit_rate.pct", "l2_hit_%"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem_%"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem_bank_conflicts"),
    ("l1tex__t_set_accesses_pipe_lsu_mem_global_op_atom.sum", "global_atomics"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum", "smem_atomic_wavefronts"),
]


def main(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        print(d["Kernel Name"][:90], f"grid={d.get('launch__grid_size')} block={d.get('launch__block_size')}")
        parts = []
        for k, name in KEYS:
            if k in d and d[k] != "":
                parts.append(f"{name}={d[k]}{'' if u.get(k) in ('', '%', None) else ' ' + u[k]}")
        print("   " + "  ".join(parts))
        st = []
        for k, v in d.items():
            if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued"):
                try:
                    st.append((float(v.replace(",", "")), k[len("smsp__pcsamp_warps_issue_stalled_"):]))
                except ValueError:
                    pass
        tot = sum(a for a, _ in st) or 1.0
        st.sort(reverse=True)
        print("   stalls: " + ", ".join(f"{n} {100 * a / tot:.0f}%" for a, n in st[:5]))


if __name__ == "__main__":
    main(sys.argv[1])
