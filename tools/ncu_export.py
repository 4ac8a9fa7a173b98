"""Compact ncu summaries for profiles/ from exported CSVs (development tool).
usage: python tools/ncu_export.py <details.csv> <raw.csv> <out.txt>"""
import csv, sys
KEYS = ['Duration', 'DRAM Throughput', 'Memory Throughput', 'L1/TEX Cache Throughput', 'L2 Cache Throughput',
        'Compute (SM) Throughput', 'Registers Per', 'Achieved Occupancy', 'Theoretical Occupancy', 'Executed Ipc A',
        'Issue Slots Busy', 'Warp Cycles Per Issued', 'L2 Hit', 'No Eligible', 'Eligible Warps', 'Executed Instructions',
        'Block Size', 'Grid Size', 'Dynamic Shared Memory Per Block']
RAW = ['dram__bytes_read.sum', 'dram__bytes_write.sum', 'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
       'sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active', 'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active',
       'smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio',
       'smsp__average_warps_issue_stalled_wait_per_issue_active.ratio',
       'smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio',
       'smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio',
       'smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio',
       'smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio', 'sm__cycles_elapsed.avg.per_second']
out = []
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[0]
for r in rows[1:]:
    if len(r) < 15:
        continue
    d = dict(zip(hdr, r))
    if any(k in d.get('Metric Name', '') for k in KEYS):
        out.append(f"{d['Kernel Name'][:44]} | {d['Section Name']} | {d['Metric Name']} | {d['Metric Unit']} | {d['Metric Value']}")
raw = list(csv.reader(open(sys.argv[2])))
units = raw[1] if len(raw) > 2 else [''] * len(raw[0])
vals = raw[2] if len(raw) > 2 else raw[1]
for k, u, v in zip(raw[0], units, vals):
    if k in RAW:
        out.append(f"raw | {k} | {u} | {v}")
open(sys.argv[3], 'w').write('\n'.join(out) + '\n')
print('\n'.join(out))
