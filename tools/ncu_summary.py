"""Key metrics of an `ncu --set full` report (one kernel launch), for profiles/.

    python tools/ncu_summary.py gpurun_out/hvp_full.ncu-rep [algorithmic_MB]
"""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__maximum_warps_per_active_cycle_pct",
        "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "launch__shared_mem_per_block_static",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "launch__grid_size",
        "launch__block_size", "smsp__inst_executed.sum", "lts__t_sector_hit_rate.pct",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"]


def main():
    rep = sys.argv[1]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for vals in rows[2:]:
        kname = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        print(f"kernel: {kname[:100]}")
        got = {}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                got[k] = (vals[i], units[i])
                print(f"  {k:60s} {vals[i]:>16s} {units[i]}")
        stalls = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued"):
                try:
                    stalls.append((float(vals[i].replace(",", "")), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        tot = sum(s for s, _ in stalls) or 1.0
        print("  stall samples: " + ", ".join(f"{n} {s / tot * 100:.1f}%" for s, n in sorted(stalls, reverse=True)[:6]))
        try:
            t_us = float(got["gpu__time_duration.sum"][0].replace(",", ""))
            tu = got["gpu__time_duration.sum"][1]
            t_us = t_us / 1000.0 if tu in ("nsecond", "ns") else t_us * (1000.0 if tu in ("msecond", "ms") else 1.0)
            # each metric carries its own unit (ncu picks Kbyte / Mbyte / Gbyte per value): scale before summing
            scale = {"Mbyte": 1.0, "Gbyte": 1e3, "Kbyte": 1e-3, "byte": 1e-6, "Tbyte": 1e6}
            mb = sum(float(got[k][0].replace(",", "")) * scale[got[k][1]]
                     for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
            print(f"  DRAM traffic {mb:.1f} MB in {t_us:.1f} us -> {mb / t_us * 1e3:.0f} GB/s (cold-cache replay)")
            if len(sys.argv) > 2:
                alg = float(sys.argv[2])
                print(f"  algorithmic {alg:.1f} MB -> {alg / t_us * 1e3:.0f} GB/s; traffic/algorithmic = {mb / alg:.3f}")
        except (KeyError, ValueError):
            pass


if __name__ == "__main__":
    main()
