"""Per-launch timeline of one call (CUDA events inside the C ABI): when each
kernel of each chunk ran, on which of the two chunk streams, and the idle
gaps.  python tools/timeline.py cfg5 [policy]"""
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_1404_0424_b200 import Context, get_config  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
ctx = Context(0)
if len(sys.argv) > 2:
    ctx.set_kernel_policy(sys.argv[2])
cfg = get_config(name)
rs = cfg.rsqrt()
rs = None if rs is None else torch.tensor(rs)
H, Y = ctx.generate_uplink(cfg.B, cfg.U, cfg.n_sc, cfg.S, cfg.seed, cfg.qam_bits, cfg.n0, rsqrt=rs)
T = ctx.generate_symbols(cfg.U, cfg.n_sc, cfg.S, cfg.seed, cfg.qam_bits) if cfg.kind == "both" else None
out = {}


def call():
    if cfg.kind == "both":
        ctx.detect_precode_cg(H, Y, cfg.rho_u, cfg.n0, cfg.es, cfg.qam_bits, cfg.K, cfg.tracker, T,
                              cfg.rho_d, cfg.K, out=out)
    else:
        ctx.detect_cg(H, Y, cfg.rho_u, cfg.n0, cfg.es, cfg.qam_bits, cfg.K, cfg.tracker, out=out)


for _ in range(3):
    call()
torch.cuda.synchronize()
ctx.set_profiling(True)
call()
torch.cuda.synchronize()
tl = ctx.kernel_timeline()
ctx.set_profiling(False)
end = max(e for _, _, e in tl)
busy = 0.0
cur_s, cur_e = None, None
for _, s, e in sorted(tl, key=lambda x: x[1]):
    if cur_e is None or s > cur_e:
        if cur_e is not None:
            busy += cur_e - cur_s
        cur_s, cur_e = s, e
    else:
        cur_e = max(cur_e, e)
busy += cur_e - cur_s
for kind, s, e in tl:
    print(f"{kind:9s} {s:8.3f} -> {e:8.3f}  ({e - s:6.3f} ms)")
print(f"span {end:.3f} ms, some kernel running {busy:.3f} ms ({100 * busy / end:.1f}%), "
      f"sum of kernel windows {sum(e - s for _, s, e in tl):.3f} ms")
