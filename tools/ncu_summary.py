"""Summarises an `ncu --set full` report for profiles/: key metrics, stall
reasons and the hottest source lines.

  python tools/ncu_summary.py gpurun_out/X.ncu-rep profiles/rNN_X.txt
"""
import csv
import io
import subprocess
import sys

sys.path.insert(0, __file__.rsplit("/", 1)[0])
import ncu_lines  # noqa: E402

KEYS = ["Kernel Name", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]


def main(rep, out):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    h, units, v = r[0], r[1], r[2]
    lines = [f"# {rep}"]
    for k in KEYS:
        if k in h:
            lines.append(f"{k}: {v[h.index(k)]} {units[h.index(k)]}".rstrip())
    stalls = [(k, float(v[i].replace(",", ""))) for i, k in enumerate(h)
              if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")
              and v[i].replace(",", "").replace(".", "").isdigit()]
    tot = sum(x for _, x in stalls) or 1
    lines.append("warp stall samples (share):")
    for k, x in sorted(stalls, key=lambda t: -t[1])[:10]:
        lines.append(f"  {k.replace('smsp__pcsamp_warps_issue_stalled_', ''):24s} {100 * x / tot:5.1f}%")
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    tmp = out + ".src.csv"
    with open(tmp, "w") as f:
        f.write(src)
    buf = io.StringIO()
    old = sys.stdout
    sys.stdout = buf
    try:
        ncu_lines.main(tmp, 25)
    finally:
        sys.stdout = old
    import os
    os.remove(tmp)
    lines.append("hottest source lines (stall-sample share, instruction share):")
    lines += ["  " + x for x in buf.getvalue().splitlines()]
    with open(out, "w") as f:
        f.write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
