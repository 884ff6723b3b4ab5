"""Shared-memory instructions with excess wavefronts (bank conflicts) in an .ncu-rep:
   python tools/ncu_conflicts.py REP [N]"""
import csv, io, subprocess, sys
out = subprocess.run(['ncu', '-i', sys.argv[1], '--page', 'source', '--csv', '--print-source', 'cuda,sass'],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if "L1 Wavefronts Shared Excessive" in r)
hdr = rows[hi]
iX, iW, iI = hdr.index("L1 Wavefronts Shared Excessive"), hdr.index("L1 Wavefronts Shared"), hdr.index("L1 Wavefronts Shared Ideal")
num = lambda x: float(x) if x.replace('.', '', 1).isdigit() else 0.0
data = [r for r in rows[hi + 1:] if len(r) > iX]
tw = sum(num(r[iW]) for r in data)
tx = sum(num(r[iX]) for r in data)
print(f"shared wavefronts {tw:.3g}, excessive {tx:.3g} ({tx / max(tw, 1) * 100:.1f}%)")
for r in sorted(data, key=lambda r: -num(r[iX]))[:int(sys.argv[2]) if len(sys.argv) > 2 else 15]:
    print(f"{num(r[iX]):12.0f} excess {num(r[iW]):12.0f} total {num(r[iI]):12.0f} ideal  {r[0][:6]:>6} {r[1][:90]}")
