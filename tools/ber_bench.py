"""Coded BLER points: GPU pipeline
(paper_1404_0424_b200.sim, one batched call per trial batch) vs the
reference's run_uplink_sweep / run_downlink_sweep on all host cores, same
seed and trials.
Prints one JSON line per config: trials/s, decoded info bits/s, BLER, and
whether the block-error counts agree.

    python tools/ber_bench.py [--trials 256] [--ref-trials 32]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))

CONFIGS = {
    # the reference SweepConfig defaults (sim.hpp:46-63) at a waterfall SNR
    "sweep_default": dict(B=32, U=8, bits=6, K=4, tracker="approx", snr=14.0, n_sc=128),
    # BASELINE config 2's array and modulation (128 x 32, 64-QAM, K = 4), 1200 subcarriers
    "cfg2_coded": dict(B=128, U=32, bits=6, K=4, tracker="approx", snr=15.0, n_sc=1200),
    # downlink: CG precoder + genie demapper (sim.cpp:205-275)
    "dl_sweep_default": dict(B=32, U=8, bits=6, K=4, snr=13.0, n_sc=128, downlink=True),
    "cfg3_coded_dl": dict(B=64, U=16, bits=6, K=4, snr=14.5, n_sc=1200, downlink=True),
}


def point(ctx, sim, c, trials, seed):
    if c.get("downlink"):
        return sim.downlink_sweep_point(ctx, c["B"], c["U"], c["bits"], c["K"], c["snr"], trials,
                                        c["n_sc"], seed)
    return sim.uplink_sweep_point(ctx, c["B"], c["U"], c["bits"], c["K"], c["tracker"], c["snr"],
                                  trials, c["n_sc"], seed)


def ref_point(ref, c, trials, seed):
    if c.get("downlink"):
        return ref.downlink_sweep_point(c["B"], c["U"], c["bits"], c["K"], c["snr"], trials,
                                        c["n_sc"], seed, threads=os.cpu_count())
    return ref.uplink_sweep_point(c["B"], c["U"], c["bits"], c["K"], c["tracker"], c["snr"],
                                  trials, c["n_sc"], seed, threads=os.cpu_count())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--trials", type=int, default=256)
    ap.add_argument("--ref-trials", type=int, default=32)
    ap.add_argument("--configs", default=",".join(CONFIGS))
    a = ap.parse_args()
    import torch
    import oracle
    from paper_1404_0424_b200 import Context, sim

    ctx = Context(0)
    ref = oracle.Oracle("ref") if oracle.available("ref") else None
    for name in a.configs.split(","):
        c = CONFIGS[name]
        # info bits per user frame (sim.cpp:38-51)
        bps = c["bits"]
        n_sym = next(s for s in range(1, 7) if (c["n_sc"] * bps * s) % 6 == 0)
        info = c["n_sc"] * bps * n_sym // 6 * 5 - 6
        point(ctx, sim, c, 8, 1)  # warm-up
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        g = point(ctx, sim, c, a.trials, 1)
        gs = time.perf_counter() - t0
        line = {"config": name, **c, "trials": a.trials, "gpu_s": round(gs, 4),
                "gpu_trials_per_s": a.trials / gs,
                "gpu_info_bits_per_s": a.trials * c["U"] * info / gs,
                "bler": g["block_errors"] / max(g["frames"], 1)}
        if ref is not None:
            rt = min(a.ref_trials, a.trials)
            t0 = time.perf_counter()
            r = ref_point(ref, c, rt, 1)
            rs = time.perf_counter() - t0
            gr = point(ctx, sim, c, rt, 1)
            line.update({"ref_trials": rt, "ref_s": round(rs, 4), "ref_threads": os.cpu_count(),
                         "ref_trials_per_s": rt / rs,
                         "speedup_trials_per_s": (a.trials / gs) / (rt / rs),
                         "block_errors_agree": gr["block_errors"] == r["block_errors"]
                         and gr["frames"] == r["frames"]})
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
