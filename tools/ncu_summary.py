"""Summarise an ncu report: SOL, occupancy, stall reasons, top SASS stall sites. python tools/ncu_summary.py rep [n]"""
import csv, io, subprocess, sys
rep = sys.argv[1]; ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 25
def run(*a):
    return subprocess.run(['ncu', '-i', rep, *a], capture_output=True, text=True).stdout
det = list(csv.reader(io.StringIO(run('--page', 'details', '--csv'))))
hdr = det[0]
want = {'Duration', 'Elapsed Cycles', 'SM Frequency', 'DRAM Throughput', 'Memory Throughput', 'L1/TEX Cache Throughput',
        'L2 Cache Throughput', 'Compute (SM) Throughput', 'Issued Ipc Active', 'Achieved Occupancy', 'Registers Per Thread',
        'Dynamic Shared Memory Per Block', 'Grid Size', 'Block Size', 'Theoretical Occupancy', 'L2 Hit Rate', 'L1/TEX Hit Rate',
        'Warp Cycles Per Issued Instruction', 'Eligible Warps Per Scheduler', 'No Eligible', 'Local Memory Spilling Requests'}
kname = None
for row in det[1:]:
    d = dict(zip(hdr, row))
    kname = d.get('Kernel Name', kname)
    if d.get('Metric Name') in want:
        print(f"{d['Metric Name']:40s} {d['Metric Value']:>14s} {d['Metric Unit']}")
print('kernel:', kname[:120] if kname else None)
raw = list(csv.reader(io.StringIO(run('--page', 'raw', '--csv'))))
for row in raw[2:]:  # one row per captured launch
    d = dict(zip(raw[0], row))
    print('== raw metrics of', d.get('Kernel Name', '?')[:100])
    for k in ['dram__bytes_read.sum', 'dram__bytes_write.sum', 'gpu__time_duration.sum',
              'smsp__sass_thread_inst_executed_op_dfma_pred_on.sum', 'smsp__sass_thread_inst_executed_op_dadd_pred_on.sum',
              'smsp__sass_thread_inst_executed_op_dmul_pred_on.sum', 'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
              'sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active', 'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum',
              'smsp__inst_executed.sum', 'sm__warps_active.avg.pct_of_peak_sustained_active']:
        if k in d: print(f'{k:60s} {d[k]} {raw[1][raw[0].index(k)]}')
    st = {k: v for k, v in d.items() if k.startswith('smsp__pcsamp_warps_issue_stalled') and not k.endswith('not_issued')}
    tot = sum(float(v.replace(',', '') or 0) for v in st.values())
    print('stall samples (share):')
    for k, v in sorted(st.items(), key=lambda kv: -float(kv[1].replace(',', '') or 0))[:10]:
        print(f'   {k.replace("smsp__pcsamp_warps_issue_stalled_", ""):28s} {float(v.replace(",", ""))/max(tot,1):6.1%}')
src = list(csv.reader(io.StringIO(run('--page', 'source', '--csv', '--print-source', 'sass'))))
h = src[1]; ix = {x: i for i, x in enumerate(h)}; rows = src[2:]
def _int(x):
    try:
        return int(x or 0)
    except ValueError:
        return 0
rows = [r for r in rows if len(r) > ix['Warp Stall Sampling (All Samples)'] and _int(r[ix['Warp Stall Sampling (All Samples)']]) >= 0 and r[ix['Address']].startswith('0x')]
tot = sum(_int(r[ix['Warp Stall Sampling (All Samples)']]) for r in rows)
print(f'top SASS stall sites ({tot} samples):')
for r in sorted(rows, key=lambda r: -_int(r[ix['Warp Stall Sampling (All Samples)']]))[:ntop]:
    print(f"  {r[ix['Address']][-5:]} {_int(r[ix['Warp Stall Sampling (All Samples)']])/max(tot,1):6.1%} exec={r[ix['Instructions Executed']]:>9s} {r[ix['Source']][:80]}")
