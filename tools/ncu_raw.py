"""Key metrics and top stall reasons of every kernel in an ncu report.

  python tools/ncu_raw.py X.ncu-rep
"""
import csv
import io
import subprocess
import sys

KEYS = ["launch__grid_size", "launch__block_size", "launch__registers_per_thread", "gpu__time_duration.sum",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_warps",
        "sm__maximum_warps_per_active_cycle_pct", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "lts__t_sectors_srcunit_tex_op_atom.sum", "lts__t_sectors_srcunit_tex_op_red.sum",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
        "lts__t_sectors_srcunit_tex_op_read.sum", "lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum",
        "lts__average_t_sector_hit_rate_srcunit_tex_op_atom.pct", "l1tex__m_xbar2l1tex_read_bytes.sum",
        "smsp__average_warp_latency_per_inst_issued.ratio", "lts__t_sectors_op_atom.sum", "lts__t_sectors_op_read.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed"]


def main(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    h, units = r[0], r[1]
    for v in r[2:]:
        print("==", v[h.index("Kernel Name")][:90])
        for k in KEYS:
            if k in h:
                print(f"  {k}: {v[h.index(k)]} {units[h.index(k)]}")
        stalls = []
        for i, k in enumerate(h):
            if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
                try:
                    stalls.append((k[len("smsp__pcsamp_warps_issue_stalled_"):], float(v[i].replace(",", ""))))
                except ValueError:
                    pass
        tot = sum(x[1] for x in stalls) or 1
        print("  stalls:", ", ".join(f"{k} {100 * x / tot:.1f}%" for k, x in sorted(stalls, key=lambda t: -t[1])[:8]))


if __name__ == "__main__":
    main(sys.argv[1])
