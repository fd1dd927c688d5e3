"""Bank model of uplink_small_kernel's full-U Gram loads (cgm_uplink_small.cuh):
lane -> (antenna part, lower 4 x 4 tile); part p reads antenna rows
p, p + KP, ... of H [B][U] (complex64, 8 U bytes per row) and takes its four
users as two 16-byte pairs in the order (01, 23) or (23, 01) (rot2).  A
quarter warp's LDS.128 is conflict-free when its lanes' 16-byte words fall in
distinct bank groups (address / 16 mod 8) or coincide.

    python tools/us_rotation.py     # wavefronts per load with / without the rotation
"""


def geometry(UP):
    nb = UP // 4
    ntile = nb * (nb + 1) // 2
    kp = 32 // ntile
    tiles = []
    rb = 0
    for t in range(ntile):
        while (rb + 1) * (rb + 2) // 2 <= t:
            rb += 1
        tiles.append((rb, t - rb * (rb + 1) // 2))
    return ntile, kp, tiles


def rot2_of(UP, part):
    """The kernel's choice (uplink_small_kernel, `rot2`)."""
    return (part >> 1) & 1 if UP == 8 else part & 1


def wavefronts(UP, rotate=True, contiguous=False, B=128):
    """Worst and mean wavefronts per quarter-warp LDS.128 over the loop's steps
    and its four loads (x pair 0 / 1, y pair 0 / 1).  contiguous=True models
    the old split (part p reads rows [pB/KP, (p+1)B/KP))."""
    ntile, kp, tiles = geometry(UP)
    worst, total, n = 0, 0, 0
    for step in range(B // kp):
        for which in range(4):  # 0: x first pair, 1: x second, 2: y first, 3: y second
            for q in range(4):
                groups = {}
                for lane in range(8 * q, 8 * q + 8):
                    part, tile = divmod(lane, ntile)
                    if part >= kp:
                        continue
                    row = part * B // kp + step if contiguous else part + kp * step
                    if row >= B:
                        continue
                    rot = rot2_of(UP, part) if rotate else 0
                    blk = tiles[tile][0] if which < 2 else tiles[tile][1]
                    pair = (which & 1) ^ rot
                    addr16 = (row * UP * 8 + (blk * 4 + 2 * pair) * 8) // 16
                    groups.setdefault(addr16 % 8, set()).add(addr16)
                w = max([len(v) for v in groups.values()] or [0])
                if w:
                    worst = max(worst, w)
                    total += w
                    n += 1
    return worst, total / max(n, 1)


if __name__ == "__main__":
    for UP in (8, 16):
        print(f"UP={UP}: rotated strided {wavefronts(UP)}, unrotated strided {wavefronts(UP, rotate=False)}, "
              f"unrotated contiguous {wavefronts(UP, rotate=False, contiguous=True)}")
