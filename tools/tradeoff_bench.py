"""The reference's complexity / performance trade-off study (sim.cpp:
475-516) end to end: one uplink sweep per
(method, iterations) over an SNR grid, then tradeoff_table at a target BLER.
GPU (paper_1404_0424_b200.sim) vs the reference's run_uplink_sweep on all
host cores with the same seeds; prints the table, both wall times and
whether every point's block errors agree.

    python tools/tradeoff_bench.py [--trials 200] [--ref-trials 200]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))

ROWS = [("chol", 1), ("cg", 2), ("cg", 3), ("cg", 4), ("cgls", 2), ("cgls", 4),
        ("neumann", 2), ("neumann", 3)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--trials", type=int, default=200)
    ap.add_argument("--ref-trials", type=int, default=200)
    ap.add_argument("--B", type=int, default=64)
    ap.add_argument("--U", type=int, default=8)
    ap.add_argument("--snr", default="8:18:1")
    a = ap.parse_args()
    import oracle
    from paper_1404_0424_b200 import Context, sim

    s0, s1, st = (float(x) for x in a.snr.split(":"))
    ctx = Context(0)
    ref = oracle.Oracle("ref") if oracle.available("ref") else None
    base = dict(bs_antennas=a.B, users=a.U, qam_bits=6, snr_start_db=s0, snr_stop_db=s1,
                snr_step_db=st, subcarriers=128, seed=1, max_breakdown_fraction=1.0)
    sim.run_sweep(ctx, sim.SweepConfig(**{**base, "trials": 4, "method": "cg", "iterations": 2}))
    t0 = time.perf_counter()
    sweeps = [sim.run_sweep(ctx, sim.SweepConfig(**base, trials=a.trials, method=m, iterations=K))
              for m, K in ROWS]
    gpu_s = time.perf_counter() - t0
    rows = sim.tradeoff_table(sweeps, 0.1)
    line = {"study": f"uplink {a.B}x{a.U} 64-QAM 128 sc, SNR {a.snr} dB, target BLER 0.1",
            "trials_per_point": a.trials, "points": sum(len(s.points) for s in sweeps),
            "gpu_s": round(gpu_s, 3),
            "table": [[r.method_label, r.iterations, r.real_mults, r.snr_db_at_target]
                      for r in rows]}
    if ref is not None:
        agree = True
        t0 = time.perf_counter()
        ref_sweeps = [ref.sweep("uplink", m, a.B, a.U, 6, K, "approx", s0, s1, st, a.ref_trials,
                                128, 1, threads=os.cpu_count()) for m, K in ROWS]
        ref_s = time.perf_counter() - t0
        diffs = []
        if a.ref_trials == a.trials:
            for (m, K), sw, rs in zip(ROWS, sweeps, ref_sweeps):
                for p, q in zip(sw.points, rs):
                    if (p.block_errors, p.frames) != (int(q["block_errors"]), int(q["frames"])):
                        agree = False
                        diffs.append([m, K, p.snr_db, p.block_errors, int(q["block_errors"]),
                                      p.frames])
        line["disagreements"] = diffs
        ref_rows = [ref.tradeoff_row(m, a.B, a.U, K, [q["snr_db"] for q in rs],
                                     [int(q["frames"]) for q in rs],
                                     [int(q["block_errors"]) for q in rs], 0.1)
                    for (m, K), rs in zip(ROWS, ref_sweeps)]
        line["ref_table"] = [[m, K, rm, snr] for (m, K), (rm, snr) in zip(ROWS, ref_rows)]
        line["table_agrees"] = all((r.real_mults, r.snr_db_at_target) == rr
                                   for r, rr in zip(rows, ref_rows))
        line.update({"ref_trials_per_point": a.ref_trials, "ref_threads": os.cpu_count(),
                     "ref_s": round(ref_s, 3),
                     "speedup_per_trial": (ref_s / a.ref_trials) / (gpu_s / a.trials),
                     "block_errors_agree": agree if a.ref_trials == a.trials else None})
    print(json.dumps(line), flush=True)
    print(sim.write_tradeoff_csv(rows, 0.1), file=sys.stderr)


if __name__ == "__main__":
    main()
