"""Per-source-line instruction counts / stall share of an .ncu-rep (needs -lineinfo):
   python tools/ncu_lines.py REP [N] [ITER_INSTR_COUNT]"""
import csv, io, subprocess, sys
out = subprocess.run(['ncu', '-i', sys.argv[1], '--page', 'source', '--csv', '--print-source', 'cuda,sass'],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[2]
iE, iS = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
num = lambda x: int(x) if x.isdigit() else 0
res = [(num(r[iE]), num(r[iS]), int(r[0]), r[1][:95]) for r in rows[3:] if r[0].isdigit()]
# normaliser: executions of the most executed barrier instruction (= per-warp iterations)
bar = max((num(r[iE]) for r in rows[3:] if len(r) > 3 and 'BAR.SYNC' in r[3]), default=1)
norm = int(sys.argv[3]) if len(sys.argv) > 3 else bar
tot, ts = sum(x[0] for x in res), sum(x[1] for x in res) or 1
print(f"instructions per warp-iteration: {tot / norm:.1f} (iterations per warp counted: {norm})")
for e, st, l, src in sorted(res, key=lambda x: -x[0])[:int(sys.argv[2]) if len(sys.argv) > 2 else 40]:
    print(f"{e / norm:6.1f} {st / ts * 100:5.1f}% L{l:4d} {src}")
