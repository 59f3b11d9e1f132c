#!/usr/bin/env python
"""Summarise an ncu report (run here, no GPU): key metrics per kernel + top stall sites.

    python tools/ncu_summary.py gpurun_out/prof_mm.ncu-rep [--source N]
"""
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.max.pct_of_peak_sustained_elapsed",
    "lts__t_sectors_srcunit_tex_op_read.sum",
    "lts__t_sectors_srcunit_tex_op_write.sum",
    "lts__t_sector_hit_rate.pct",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "launch__grid_size",
    "launch__registers_per_thread",
]


def ncu(args):
    return subprocess.run(["ncu", *args], capture_output=True, text=True).stdout


def main():
    rep = sys.argv[1]
    nsrc = int(sys.argv[sys.argv.index("--source") + 1]) if "--source" in sys.argv else 0
    rows = list(csv.reader(io.StringIO(ncu(["-i", rep, "--page", "raw", "--csv"]))))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")][:60]
        print(f"== [{r[0]}] {name}")
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                print(f"   {k:80s} {r[i]:>14s} {units[i]}")
    if nsrc:
        for kid in range(len(rows) - 2):
            src = list(csv.reader(io.StringIO(ncu(["-i", rep, "--page", "source", "--csv", "--launch-skip",
                                                   str(kid), "--launch-count", "1"]))))
            h = src[1]
            data = src[2:]
            i_s = h.index("Warp Stall Sampling (All Samples)")
            i_e = h.index("Instructions Executed")
            tot = sum(int(x[i_s]) for x in data if x[i_s].isdigit())
            print(f"== source [{kid}] samples {tot}")
            for x in sorted(data, key=lambda x: -int(x[i_s]) if x[i_s].isdigit() else 0)[:nsrc]:
                print(f"   {x[i_s]:>6s} {x[i_e]:>9s} {x[0][-5:]} {x[1][:90]}")


if __name__ == "__main__":
    main()
