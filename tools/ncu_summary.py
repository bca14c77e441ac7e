"""Summarise .ncu-rep captures into the JSON kept under profiles/.

    python tools/ncu_summary.py out.json name=gpurun_out/x.ncu-rep [name2=gpurun_out/ncu/y.raw.csv ...]
"""
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__bytes.sum.per_second",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum",
    "lts__t_sector_hit_rate.pct",
    "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__cycles_elapsed.avg.per_second",
    "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic",
    "launch__grid_size",
    "launch__cluster_dim_x",
]


def summarise(rep):
    if rep.endswith(".csv"):  # a `--page raw --csv` export made on the GPU box (tools/prof_all.sh)
        out = open(rep).read()
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head, units, vals = rows[0], rows[1], rows[2]
    res = {"kernel": vals[head.index("Kernel Name")]}
    for k in KEYS:
        if k in head:
            i = head.index(k)
            res[k] = f"{vals[i]} {units[i]}".strip()
    return res


def main():
    dst = sys.argv[1]
    try:
        data = json.load(open(dst))
    except FileNotFoundError:
        data = {}
    for arg in sys.argv[2:]:
        name, rep = arg.split("=", 1)
        data[name] = summarise(rep)
    json.dump(data, open(dst, "w"), indent=1)
    print(json.dumps(data, indent=1))


if __name__ == "__main__":
    main()
