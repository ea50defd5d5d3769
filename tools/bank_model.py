"""Shared-memory bank-conflict model of the CG line kernel's transposes (development aid).

    python tools/bank_model.py [N] [C]

Element (i0, i1, i2) of a cell buffer sits at word i0*A + i1*B + i2*S (+ cell * CS); a
warp's 64-bit access takes max_j #{distinct words w with w % 16 == j} wavefronts (16
double-banks of 8 B).  Counts the wavefronts of the 23 line accesses of cell_laplace
(8 z-pattern, 9 y-pattern, 6 x-pattern) for the block layout (N^2 threads x C cells)
and searches paddings B = N + pb, S = B*N + ps and the cell stride.
"""
import itertools
import sys

N = int(sys.argv[1]) if len(sys.argv) > 1 else 5
C = int(sys.argv[2]) if len(sys.argv) > 2 else 8
N2 = N * N
THREADS = N2 * C
ACC = {"z": 8, "y": 9, "x": 6}


def wavefronts(words):
    cnt = {}
    for w in set(words):
        cnt[w % 16] = cnt.get(w % 16, 0) + 1
    return max(2 if len(words) > 16 else 1, max(cnt.values()))


def cost(A, B, S, CS):
    tot = {}
    for pat in ("z", "y", "x"):
        wf = 0
        for w0 in range(0, THREADS, 32):
            for l in range(N):
                words = []
                for tid in range(w0, min(w0 + 32, THREADS)):
                    t, ci = tid % N2, tid // N2
                    ta, tb = t % N, t // N
                    i0, i1, i2 = {"z": (ta, tb, l), "y": (ta, l, tb), "x": (l, ta, tb)}[pat]
                    words.append(ci * CS + i0 * A + i1 * B + i2 * S)
                wf += wavefronts(words)
        tot[pat] = wf
    return sum(ACC[p] * tot[p] for p in tot), tot


def ideal():
    return sum(ACC.values()) * sum(N * (2 if min(32, THREADS - w0) > 16 else 1) for w0 in range(0, THREADS, 32))


base = cost(1, N, N2, 3 * N * N * N + (2 if N == 5 else 0))
print(f"N={N} C={C} ideal {ideal()}  current {base}")
best = []
for pb in range(0, 4):
    for ps in range(0, 8):
        B = N + pb
        S = B * N + ps
        field = (N - 1) * (1 + B + S) + 1
        for cp in range(0, 17):
            CS = 3 * field + cp
            c, d = cost(1, B, S, CS)
            best.append((c, pb, ps, cp, CS, d))
best.sort()
for b in best[:10]:
    print(b)
