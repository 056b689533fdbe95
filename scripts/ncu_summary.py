"""Summarise one ncu --set full capture (.ncu-rep): key raw counters, DRAM
traffic per system, stall mix and the SASS segment attribution.
usage: python scripts/ncu_summary.py rep.ncu-rep systems_in_capture [systems_per_bench_launch]"""
import csv
import io
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "launch__grid_size", "launch__block_size",
        "launch__registers_per_thread", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "sm__cycles_elapsed.avg"]


def main(rep, nsys, nbench=4096):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    d = dict(zip(rows[0], rows[2]))
    u = dict(zip(rows[0], rows[1]))
    for k in KEYS:
        print(f"{k} {d.get(k)} {u.get(k, '')}")

    def mbytes(k):
        v = float(d[k].replace(",", ""))
        return v * {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}[u[k]]
    traffic_mb = mbytes("dram__bytes_read.sum") + mbytes("dram__bytes_write.sum")
    print(f"dram traffic per system {traffic_mb * 1e6 / nsys / 1e3:.1f} KB; scaled to a {nbench}-system "
          f"launch {traffic_mb * 1e6 / nsys * nbench:.4g} B")
    samp = {k: float(v.replace(",", "")) for k, v in d.items()
            if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued") and v}
    tot = sum(samp.values()) or 1
    for k, v in sorted(samp.items(), key=lambda x: -x[1])[:10]:
        print(f"{100 * v / tot:5.1f}% {k.replace('smsp__pcsamp_warps_issue_stalled_', '')}")
    return traffic_mb * 1e6 / nsys * nbench


if __name__ == "__main__":
    t = main(sys.argv[1], int(sys.argv[2]), int(sys.argv[3]) if len(sys.argv) > 3 else 4096)
