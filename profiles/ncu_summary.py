"""Summarise every kernel of an ncu report: python profiles/ncu_summary.py <report.ncu-rep>."""
import csv
import subprocess
import sys

WANT = ['Kernel Name', 'gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'lts__t_sector_hit_rate.pct',
        'l1tex__t_sector_hit_rate.pct', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'launch__registers_per_thread', 'launch__occupancy_limit_registers', 'launch__occupancy_limit_shared_mem',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed', 'lts__throughput.avg.pct_of_peak_sustained_elapsed',
        'l1tex__throughput.avg.pct_of_peak_sustained_elapsed', 'launch__grid_size',
        'lts__t_sectors_srcunit_tex_op_read.sum', 'lts__t_requests_srcunit_tex_op_read.sum', 'smsp__inst_executed.sum',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum', 'l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum',
        'l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum']

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, units = rows[0], rows[1]
for vals in rows[2:]:
    for w in WANT:
        for i, h in enumerate(hdr):
            if h == w:
                print(f"{w:60s} {units[i]:>10s} {vals[i]}")
    for i, h in enumerate(hdr):
        if 'average_warps_issue_stalled' in h and h.endswith('per_issue_active.ratio'):
            try:
                v = float(vals[i])
            except ValueError:
                continue
            if v > 0.3:
                print(f"{h:60s} {v}")
    print()
