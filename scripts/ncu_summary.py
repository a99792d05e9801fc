"""Summarise an ncu --set full report: key throughput, occupancy and stall
metrics (per kernel row). Usage: python scripts/ncu_summary.py report.ncu-rep"""
import csv
import io
import re
import subprocess
import sys

PAT = re.compile(
    r"^(gpu__time_duration.sum|dram__bytes_(read|write)\.sum|dram__throughput.avg.pct_of_peak_sustained_elapsed|"
    r"sm__throughput.avg.pct_of_peak_sustained_elapsed|launch__registers_per_thread|"
    r"sm__warps_active.avg.pct_of_peak_sustained_active|lts__t_sector_hit_rate.pct|"
    r"l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_(ld|st).sum|sm__inst_executed_pipe_fp64.sum|"
    r"sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active|smsp__issue_active.avg.pct_of_peak_sustained_active|"
    r"lts__t_sectors_srcunit_tex_op_(read|write).sum|launch__grid_size|launch__occupancy_limit_registers|"
    r"smsp__average_warps_issue_stalled_[a-z_]+_per_issue_active.ratio)$")


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for vals in rows[2:]:
        d = dict(zip(hdr, vals))
        print("==", d.get("Kernel Name", "?")[:120])
        stalls = []
        for k, u in zip(hdr, units):
            if PAT.match(k):
                if k.startswith("smsp__average_warps_issue_stalled"):
                    try:
                        stalls.append((float(d[k]), k))
                    except ValueError:
                        pass
                else:
                    print(f"  {k} = {d[k]} {u}")
        for v, k in sorted(stalls, reverse=True)[:8]:
            print(f"  stall {k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')} = {v:.3f}")


if __name__ == "__main__":
    main(sys.argv[1])
