"""Key metrics + stall breakdown from an ncu report.  Usage: ncu_summary.py report.ncu-rep"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
keep = ['Duration', 'Executed Ipc Active', 'Issue Slots Busy', 'Executed Instructions', 'No Eligible',
        'Eligible Warps Per Scheduler', 'Achieved Occupancy', 'Registers Per Thread',
        'Dynamic Shared Memory Per Block', 'Theoretical Occupancy', 'Warp Cycles Per Issued Instruction',
        'Compute (SM) Throughput', 'DRAM Throughput', 'SM Frequency', 'Grid Size']
r = csv.reader(io.StringIO(det))
hdr = next(r)
for row in r:
    d = dict(zip(hdr, row))
    if d.get('Metric Name') in keep:
        print(d['Metric Name'].ljust(40), d['Metric Value'], d['Metric Unit'])
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, vals = rows[0], rows[2] if len(rows) > 2 else rows[1]
d = dict(zip(hdr, vals))
def num(v):
    try:
        return float(v.replace(',', ''))
    except Exception:
        return None
items = [(k.replace('smsp__pcsamp_warps_issue_stalled_', ''), num(v)) for k, v in d.items()
         if k.startswith('smsp__pcsamp_warps_issue_stalled_') and not k.endswith('not_issued') and num(v) is not None]
tot = sum(v for _, v in items) or 1
print('stalls:', ', '.join(f'{k} {100*v/tot:.1f}%' for k, v in sorted(items, key=lambda kv: -kv[1])[:9]))
for k in ['sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active',
          'sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active',
          'sm__inst_executed_pipe_fmaheavy.avg.pct_of_peak_sustained_active',
          'sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active',
          'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active',
          'dram__bytes_read.sum', 'dram__bytes_write.sum', 'gpu__time_duration.sum']:
    if k in d:
        print(k.ljust(64), d[k])
