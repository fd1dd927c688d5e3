import sys, torch
sys.path.insert(0, '.')
from paper_1404_0424_b200 import Context
ctx = Context(0)
for U, B in [(4, 16), (8, 32), (16, 64), (32,128)]:
    for n_sc in (37, 6144):
        for S in (1, 2, 3):
            for K in (1, 2, 4):
                g = torch.Generator().manual_seed(U)
                H = torch.complex(torch.randn(n_sc, B, U, generator=g), torch.randn(n_sc, B, U, generator=g)).cuda() / 2**0.5
                T = torch.complex(torch.randn(n_sc, S, U, generator=g), torch.randn(n_sc, S, U, generator=g)).cuda() / 2**0.5
                Hd = H.conj().transpose(1, 2).contiguous()
                a = ctx.precode_cg(H, T, 3.0, K, uplink_layout=True)
                b = ctx.precode_cg(Hd, T, 3.0, K)
                torch.cuda.synchronize()
                d = float((a["s"] - b["s"]).abs().max())
                print(U, B, n_sc, S, K, f"{d:.2e}", "BAD" if d > 1e-4 else "")
