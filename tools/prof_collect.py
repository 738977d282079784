"""Writes the round's profiles/ from a tools/prof_refresh.sh run (gpurun_out/):
ncu summaries per kernel, the bench launch list, the bench line, per-config
probe numbers, and profiles/traffic.json (DRAM bytes and warp instructions of
the bench's executor launch, read by bench.py).

  python tools/prof_collect.py r01
"""
import csv
import io
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
import ncu_summary  # noqa: E402

G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    return dict(zip(r[0], r[2])), dict(zip(r[0], r[1]))


def num(v):
    return float(v.replace(",", ""))


def main(tag):
    reps = {"redrec_full": "redrec_kernel_full", "plan_full": "redrec_plan_kernel_full",
            "bird_full": "bird_kernel_full", "chain_full": "chain_band_kernel_full",
            "c3_batch_full": "c3_batch_pipeline_kernel_full"}
    for rep, name in reps.items():
        f = os.path.join(G, rep + ".ncu-rep")
        if os.path.exists(f):
            ncu_summary.main(f, os.path.join(P, f"{tag}_{name}.txt"))
            print("wrote", name)
    for src, dst in (("launches.csv", "launches_bench.csv"), ("c3_launches.csv", "launches_c3_pipeline.csv"),
                     ("probe_all.jsonl", "probe_all.jsonl")):
        if os.path.exists(os.path.join(G, src)):
            shutil.copy(os.path.join(G, src), os.path.join(P, f"{tag}_{dst}"))
    bj = os.path.join(G, "bench.json")
    if os.path.exists(bj):
        lines = [x for x in open(bj).read().splitlines() if x.startswith("{")]
        if lines:
            open(os.path.join(P, f"{tag}_bench_b200.json"), "w").write(lines[-1] + "\n")
    f = os.path.join(G, "redrec_full.ncu-rep")
    if os.path.exists(f):
        v, u = raw(f)
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        rd = num(v["dram__bytes_read.sum"]) * scale[u["dram__bytes_read.sum"]]
        wr = num(v["dram__bytes_write.sum"]) * scale[u["dram__bytes_write.sum"]]
        tr = {"_source": "ncu --set full --clock-control none on `python bench.py --steps 1 --warmup 3 --no-cpu`, "
                         "launch 4 of redrec_kernel (after 3 warm-ups): dram__bytes_read.sum + dram__bytes_write.sum "
                         f"and smsp__inst_executed.sum of that launch; summary in profiles/{tag}_redrec_kernel_full.txt",
              "redrec_kernel": {"batch": 2048, "workload_seed": "0x25600000", "dram_bytes": int(rd + wr),
                                "dram_read": int(rd), "dram_write": int(wr),
                                "warp_inst": int(num(v["smsp__inst_executed.sum"]))}}
        json.dump(tr, open(os.path.join(P, "traffic.json"), "w"), indent=1)
        print("wrote traffic.json", tr["redrec_kernel"])


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r01")
