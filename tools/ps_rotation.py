"""Search the per-lane start rotation of precode_small_kernel's Gram loads
(U = 16: 10 lower 4x4 tiles x 3 antenna-pair ranges of a 64-antenna chunk)
so that every quarter-warp LDS.128 phase hits distinct 16-byte bank groups.
Row stride 66 float2 = 33 x 16 B; bank group = (33 row + pair) mod 8.

    python tools/ps_rotation.py
"""
import random

NTILE, KP, NP, LD16 = 10, 3, 32, 33
tiles = []
rb = 0
for t in range(NTILE):
    while (rb + 1) * (rb + 2) // 2 <= t:
        rb += 1
    tiles.append((rb, t - rb * (rb + 1) // 2))
lanes = []
for lane in range(32):
    part, tile = divmod(lane, NTILE)
    if part >= KP:
        lanes.append(None)
        continue
    q0 = part * NP // KP
    lanes.append((tiles[tile][0], tiles[tile][1], q0, (part + 1) * NP // KP - q0, tile))


def cost(rot):
    tot = 0
    for it in range(11):
        for ph in range(4):
            for which in (0, 1):
                groups = {}
                for lane in range(ph * 8, ph * 8 + 8):
                    L = lanes[lane]
                    if L is None or it >= L[3] or (which == 1 and L[0] == L[1]):
                        continue
                    q = L[2] + (rot[lane] + it) % L[3]
                    addr = 4 * (L[0] if which == 0 else L[1]) * LD16 + q
                    groups.setdefault(addr % 8, set()).add(addr)
                tot += max([len(v) for v in groups.values()] or [0])
    return tot


base = [(L[4] % L[3]) if L else 0 for L in lanes]
best, bc = base[:], cost(base)
print("tile mod range:", bc)
random.seed(1)
for _ in range(20000):
    c = best[:]
    l = random.randrange(30)
    c[l] = random.randrange(lanes[l][3])
    cc = cost(c)
    if cc <= bc:
        best, bc = c, cc
print("searched:", bc, best)
