"""Opcode histogram (executed warp-instructions and stall share) of an ncu report: python tools/ncu_ops.py rep [n]"""
import collections, csv, io, subprocess, sys
rep = sys.argv[1]; n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass'], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out))); h = rows[1]; ix = {x: i for i, x in enumerate(h)}
cnt = collections.Counter(); st = collections.Counter()
for r in rows[2:]:
    src = r[ix['Source']].strip()
    toks = src.split()
    if not toks: continue
    op = toks[1] if toks[0].startswith('@') and len(toks) > 1 else toks[0]
    op = op.split('.')[0]
    cnt[op] += int(r[ix['Instructions Executed']] or 0)
    st[op] += int(r[ix['Warp Stall Sampling (All Samples)']] or 0)
tot = sum(cnt.values()); ts = sum(st.values()) or 1
for op, c in cnt.most_common(n):
    print(f'{op:10s} {c:>12d} {c/tot:6.1%}  stall {st[op]/ts:6.1%}')
print('total', tot)
