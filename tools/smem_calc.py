"""SMEM footprint of a zwave variant (mirrors ZwaveConfig in zwave.cuh)."""
import sys
RAD = {0: 1, 1: 1, 2: 4, 3: 4}
NAUXA = {0: 0, 1: 7, 2: 2, 3: 13}
r16 = lambda n: (n + 15) // 16 * 16


def smem(kind, tb, lx, ly, nt, p, pa):
    R = RAD[kind]; QL = R + 1; NR0 = R + 1 + p; H = tb * R
    OY = ly - 2 * H; OXM = lx - 2 * H; CELLS = lx * ly
    NRING = NR0 + (tb - 1) * QL
    NAUX = NAUXA[kind]; AXO = R & ~1; AX = lx - 2 * AXO; AY = ly - 2 * R
    NAR = ((1 if (kind == 1 and tb == 2) else (tb - 1) * R + 1) + pa) if NAUX else 0
    AUXPLANE = NAUX * AX * AY
    GUARD = r16(lx * R + R + 8); STAGE = r16(OXM * OY)
    d = 2 * GUARD + NRING * CELLS + NAR * AUXPLANE + 3 * STAGE
    return d * 8 + 8 * (NR0 + NAR)


if __name__ == "__main__":
    for line in sys.stdin:
        a = [int(x) for x in line.replace(",", " ").split()[:7]]
        b = smem(*a)
        print(a, b, f"{b/1024:.1f}KB", "OK" if b <= 232448 else "TOO BIG", "per-SM CTAs by smem:", 233472 // (b + 1024))
