"""Summarise an `ncu --set full` report of the conv kernels for profiles/.

usage: python tools/ncu_summary.py report.ncu-rep images_per_launch out_prefix
writes <out_prefix>.txt (per-kernel key metrics) and profiles/ncu_traffic.json (DRAM bytes per
launch by layer, read by bench.py for roofline.traffic).
"""
import csv
import io
import json
import os
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "launch__grid_size", "launch__block_size",
        "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_bytes.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum"]
LAYER_OF = {"conv_first_lp_kernel": "layer0", "conv_strip_kernel": "layer0", "conv_patch_kernel": "layer0",
            "conv_first_tc_kernel": "layer0", "conv_first_tc_pool_kernel": "layer0",
            "conv_first_tma_pool_kernel": "layer0", "conv1_fp4_pool_kernel": "layer0", "conv_bin_kernel": "layer1", "conv_tc_kernel": "layer1",
            "conv_tc4_kernel": "layer1", "conv_tc4_pool_kernel": "layer1", "conv_tc4_pool3_kernel": "layer1", "dense_kernel": "layer2",
            "dense_tc4_kernel": "layer2"}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main():
    rep, imgs, prefix = sys.argv[1], int(sys.argv[2]), sys.argv[3]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    ki = hdr.index("Kernel Name")
    lines, traffic = [], {}
    tfile = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "ncu_traffic.json")
    if os.path.exists(tfile):
        traffic = json.load(open(tfile))
    for r in rows[2:]:
        name = r[ki]
        lines.append(name)
        vals = {}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                lines.append("    %-62s %s %s" % (k, r[i], units[i]))
                vals[k] = (r[i], units[i])
        short = name.split("<")[0].replace("void ", "").replace("bnn::", "")
        if short in LAYER_OF and "dram__bytes_read.sum" in vals:
            b = sum(float(vals[k][0].replace(",", "")) * SCALE.get(vals[k][1], 1)
                    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
            traffic[LAYER_OF[short]] = {"kernel": name, "dram_bytes_per_launch": b, "images_per_launch": imgs,
                                        "source": os.path.basename(rep)}
    open(prefix + ".txt", "w").write("\n".join(lines) + "\n")
    json.dump(traffic, open(tfile, "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
