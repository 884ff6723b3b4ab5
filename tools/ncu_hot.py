"""Top stalled SASS instructions of an .ncu-rep (source page):  python tools/ncu_hot.py REP [N]"""
import csv, io, subprocess, sys
out = subprocess.run(['ncu', '-i', sys.argv[1], '--page', 'source', '--csv', '--print-source', 'sass'],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, data = rows[1], rows[2:]
iS, iSrc, iE = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Source"), hdr.index("Instructions Executed")
cols = [i for i, h in enumerate(hdr) if h.startswith('stall_') and 'Not Issued' not in h]
tot = sum(int(r[iS]) for r in data)
print("samples", tot, "instructions", len(data))
for r in sorted(data, key=lambda r: -int(r[iS]))[:int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    st = sorted(((hdr[i][6:], int(r[i])) for i in cols if r[i] not in ('0', '', '-')), key=lambda x: -x[1])[:3]
    print(f"{int(r[iS]) / tot * 100:5.1f}% {r[0][-5:]} {r[iE]:>9} {r[iSrc].strip()[:58]:58s} {dict(st)}")
