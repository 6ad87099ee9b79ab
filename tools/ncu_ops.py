"""Executed warp-instructions by SASS opcode from an ncu report: python tools/ncu_ops.py rep [n]"""
import csv, io, subprocess, sys
from collections import Counter
rep = sys.argv[1]; n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass'], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]; ix = {x: i for i, x in enumerate(h)}
ops = Counter(); tot = 0
for r in rows[2:]:
    try: e = int(r[ix['Instructions Executed']] or 0)
    except ValueError: continue
    src = r[ix['Source']].strip()
    op = src.split()[0] if src else '?'
    if op.startswith('@'): op = src.split()[1]
    ops[op.split('.')[0]] += e; tot += e
print('total', tot)
for op, e in ops.most_common(n): print(f'{op:12s} {e/1e9:8.3f} G  {100*e/tot:5.1f}%')
