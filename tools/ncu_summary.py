"""Summarize an ncu --set full capture (raw page CSV) into the JSON kept under profiles/.

    python tools/ncu_summary.py <report.ncu-rep | raw.csv> <out.json> "<capture command>"
"""
import csv
import json
import os
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__ops_path_tensor_op_utcimma_src_int8_sparsity_off.sum.pct_of_peak_sustained_elapsed",
    "sm__ops_path_tensor_op_utchmma_src_fp16_dst_fp32_sparsity_off.sum.pct_of_peak_sustained_elapsed",
    "sm__ops_path_tensor_op_utcqmma_src_fp4_fp6_fp8_dst_fp32_sparsity_off.sum.pct_of_peak_sustained_elapsed",
    "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
    "lts__t_sector_hit_rate.pct", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__m_xbar2l1tex_read_bytes.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__block_size",
]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def main():
    src, out, cmd = sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else ""
    if src.endswith(".ncu-rep"):
        text = subprocess.run(["ncu", "-i", src, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    else:
        text = open(src).read()
    rows = list(csv.reader(text.splitlines()))
    h, u, v = rows[0], rows[1], rows[2]
    idx = {k: i for i, k in enumerate(h)}
    met = {k: f"{v[idx[k]]} {u[idx[k]]}".strip() for k in KEYS if k in idx}
    def nbytes(k):
        i = idx.get(k)
        return float(v[i].replace(",", "")) * SCALE.get(u[i], 1) if i is not None else None
    rd, wr = nbytes("dram__bytes_read.sum"), nbytes("dram__bytes_write.sum")
    res = {"capture": cmd, "kernel": v[idx["Kernel Name"]] if "Kernel Name" in idx else None, "metrics": met,
           "dram_read_bytes": rd, "dram_write_bytes": wr,
           "dram_bytes_per_launch": (rd + wr) if rd is not None and wr is not None else None}
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
