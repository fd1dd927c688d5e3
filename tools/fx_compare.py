"""fx (fused basis + extraction) vs materialised basis, per K: max |mu| / |rho| differences."""
import os, sys, torch
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_1404_0424_b200 import Context
ctx = Context(0)
for U, B in ((32, 64), (64, 128)):
    g = torch.Generator().manual_seed(U)
    n_sc = 600
    H = torch.complex(torch.randn(n_sc, B, U, generator=g), torch.randn(n_sc, B, U, generator=g)).cuda() / 2 ** 0.5
    Y = torch.complex(torch.randn(n_sc, B, 1, generator=g), torch.randn(n_sc, B, 1, generator=g)).cuda()
    for K in (1, 2, 3, 4, 8):
        os.environ.pop("CGMIMO_FX", None)
        a = ctx.detect_cg(H, Y, 3.0, 0.3, 1.0, 6, K, "exact")
        os.environ["CGMIMO_FX"] = "0"
        b = ctx.detect_cg(H, Y, 3.0, 0.3, 1.0, 6, K, "exact")
        torch.cuda.synchronize()
        print(U, K, {k: float((a[k] - b[k]).abs().max()) for k in ("xhat", "mu", "rho")}, float(b["mu"].abs().mean()))
    os.environ.pop("CGMIMO_FX", None)
