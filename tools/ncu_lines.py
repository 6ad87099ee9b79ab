"""Stall samples and executed instructions per CUDA source line: python tools/ncu_lines.py rep [n]"""
import csv, io, subprocess, sys
rep = sys.argv[1]; n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'cuda,sass'],
                     capture_output=True, text=True).stdout
cur = None; hdr = None; res = []
for r in csv.reader(io.StringIO(out)):
    if len(r) == 2 and r[0] == 'File Path': cur = r[1].split('/')[-1]; continue
    if r and r[0] == 'Line No': hdr = {x: i for i, x in enumerate(r)}; continue
    if hdr and r and r[0].isdigit():
        try:
            s = int(r[4] or 0); e = int(r[7] or 0)
        except ValueError:
            continue
        res.append((s, e, cur, int(r[0]), r[1].strip()[:90]))
tot = sum(x[0] for x in res) or 1; te = sum(x[1] for x in res) or 1
print(f'samples {tot} warp-inst {te}')
for s, e, f, l, src in sorted(res, reverse=True)[:n]:
    print(f'{100 * s / tot:5.1f}% stall {100 * e / te:5.1f}% inst  {f}:{l}  {src}')
