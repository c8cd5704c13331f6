"""One line per captured kernel from ncu reports (--page raw --csv):
duration, DRAM traffic and bandwidth, L2 hit, L2/SM/tensor throughput.

    python tools/summarize_ncu.py gpurun_out/prof_*.ncu-rep > profiles/r01/ncu_kernels_summary.txt
"""

import csv
import io
import subprocess
import sys

METRICS = {
    "dur_ms": "gpu__time_duration.sum",
    "dram_rd_GB": "dram__bytes_read.sum",
    "dram_wr_GB": "dram__bytes_write.sum",
    "dram_pct": "FBSP.TriageCompute.dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "l2_hit_pct": "lts__t_sector_hit_rate.pct",
    "l2_pct": "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "tensor_pct": "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "smem_tc_pct": "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "warps_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
}
SCALE = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "second": 1e3,
         "s": 1e3, "byte": 1e-9, "Kbyte": 1e-6, "KB": 1e-6, "Mbyte": 1e-3, "MB": 1e-3, "Gbyte": 1.0, "GB": 1.0,
         "Tbyte": 1e3, "TB": 1e3}


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    if len(r) < 3:
        return []
    head, units = r[0], r[1]
    res = []
    for row in r[2:]:
        d = {}
        for key, m in METRICS.items():
            if m in head:
                i = head.index(m)
                try:
                    v = float(row[i].replace(",", ""))
                except ValueError:
                    continue
                d[key] = v * SCALE.get(units[i], 1.0)
        name = row[head.index("Kernel Name")] if "Kernel Name" in head else "?"
        res.append((name.split("(")[0][:70], d))
    return res


def main():
    keys = list(METRICS)
    print("# " + " | ".join(["kernel"] + keys + ["dram_GBps"]) + "  (report)")
    for rep in sys.argv[1:]:
        for name, d in rows(rep):
            gbps = (d.get("dram_rd_GB", 0) + d.get("dram_wr_GB", 0)) / (d["dur_ms"] * 1e-3) if d.get("dur_ms") else 0
            vals = [f"{d[k]:.3f}" if k in d else "-" for k in keys]
            print(" | ".join([name] + vals + [f"{gbps:.0f}"]) + f"  ({rep.split('/')[-1]})")


if __name__ == "__main__":
    main()
