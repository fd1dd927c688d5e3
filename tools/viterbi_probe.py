import sys, torch, numpy as np
sys.path.insert(0, '.')
from paper_1404_0424_b200 import Context
ctx = Context(0)
rng = np.random.default_rng(0)
llr = rng.standard_normal((2048, 7200)) * 3
ctx.viterbi_decode(llr[:16])
import time; t=time.perf_counter(); ctx.viterbi_decode(llr); print("2048 cw", time.perf_counter()-t)
