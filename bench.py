"""bench.py -- throughput of the B200 CG detection + precoding path on
BASELINE's multi-GPU workload (configs[4] = cfg5: B=256, U=32, correlated
channel, exact SINR, K=4, 64-QAM, then CG precoding on the same channels;
65,536 subcarriers x 16 symbols = 1,048,576 instances split over the GPUs).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config cfg5]

* a step = one pass of the hot path (channel -> moments -> solve -> precoder
  kernels, through the C ABI) over the rank's shard of the job with inputs
  resident in HBM (6.4 GB of H + Y per GPU at N = 1, far above the 126 MB L2);
* value = whole-job vectors/s (max device time over ranks, CUDA events on the
  launching stream); e2e = the same metric through the public host-buffer
  API (pinned host H/Y/T in, every output out, copies in the timed region);
* N > 1 (torchrun): strong scaling, rank r takes shard_range(65536, r, N); no
  data-path collective; the whole job with the chunked, overlapped gather of
  LLRs + precoded vectors to rank 0 (cgm_gatherv, NCCL) is timed separately
  and reported under "gather" with its NVLink roofline term;
* other configs (--config cfg1..cfg4b) are weak-scaling parity/bench cases;
* --impl reference: the unmodified reference (oracle/_ref, FP64 per-call
  detect_cg + precode_cg over all host threads) on a >= 10 s subsample of the
  same workload and the same input values, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "detected subcarrier-vectors/s"
UNIT = "vectors/s"


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    peaks = {"hbm_gbs": 6449.1, "sm_max_mhz": 1965.0, "source": "fallback"}
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        peaks.update({k: d[k] for k in ("hbm_gbs", "sm_max_mhz") if k in d})
        peaks["source"] = "MEASURED_PEAKS.json"
    return peaks


class ClockSampler:
    """NVML sampling of SM clock + throttle reasons while the timed region runs."""

    def __init__(self, device: int, period_s: float = 0.002):
        self.device = device
        self.period = period_s
        self.samples = []
        self.reasons = set()
        self._stop = threading.Event()
        self._t = None
        self.max_mhz = None

    def __enter__(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            names = {
                "hw_slowdown": getattr(pynvml, "nvmlClocksThrottleReasonHwSlowdown", 0x8),
                "hw_thermal_slowdown": getattr(pynvml, "nvmlClocksThrottleReasonHwThermalSlowdown", 0x40),
                "sw_thermal_slowdown": getattr(pynvml, "nvmlClocksThrottleReasonSwThermalSlowdown", 0x20),
                "sw_power_cap": getattr(pynvml, "nvmlClocksThrottleReasonSwPowerCap", 0x4),
                "hw_power_brake_slowdown": getattr(pynvml, "nvmlClocksThrottleReasonHwPowerBrakeSlowdown", 0x80),
            }

            def run():
                while not self._stop.is_set():
                    try:
                        self.samples.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                        r = pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                        for n, bit in names.items():
                            if r & bit:
                                self.reasons.add(n)
                    except Exception:
                        pass
                    time.sleep(self.period)

            self._t = threading.Thread(target=run, daemon=True)
            self._t.start()
        except Exception as e:  # NVML unavailable: record why
            self.reasons.add(f"nvml-unavailable:{type(e).__name__}")
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=1)

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "samples": len(self.samples),
                "reasons": sorted(self.reasons)}


def read_traffic(cfg_name: str):
    """dram bytes (read + write) per launch of each kernel, from the committed
    ncu --set full capture: {"channel": B, "solve": B} or None."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        v = json.load(f).get(cfg_name)
    return v if isinstance(v, dict) else None


# a stated subsample of >= 10 s of CPU work (the CPU tests of the
# JSON contract shorten it through BENCH_CPU_MIN_SECONDS)
CPU_MIN_SECONDS = float(os.environ.get("BENCH_CPU_MIN_SECONDS", "10.0"))


def cpu_reference(cfg_name: str) -> dict:
    """The unmodified reference (oracle/_ref, FP64 per-call API over all host
    threads) on a subsample of the workload that takes >= 10 s per pass, best
    of 3 passes (the calibration pass is the warm-up), rate extrapolated
    linearly; inputs are the GPU arm's own complex64 values (subcarriers
    0..n-1 of its frame 0), re-drawn on the host from the same seeded streams."""
    import oracle.cpu_bench as cb

    return cb.spawn(cfg_name, 1, os.cpu_count() or 1, passes=3, warmup=0, timeout=1800,
                    min_seconds=CPU_MIN_SECONDS)


def reference_arm(args, rank, world):
    if rank != 0:
        return
    from paper_1404_0424_b200.configs import get_config

    cfg = get_config(args.config)
    r = cpu_reference(args.config)
    v = r["value"]
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": cfg.vectors / v * 1e3,  # one whole-config step at the sampled rate
        "higher_is_better": True, "scaling": "strong" if cfg.name == "cfg5" else "weak", "vs_baseline": None, "dtype": "complex128",
        "data": "synthetic", "config": workload_config(cfg, world=world),
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": r["cores"], "kind": r["kind"],
                         "sample": r["sample"]},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "llr_gbit_s": v * cfg.U * cfg.qam_bits / 1e9,
    }
    print(json.dumps(line), flush=True)


def workload_config(cfg, frames=None, world=1):
    strong = cfg.name == "cfg5"
    d = {"workload": f"{cfg.name}: {cfg.kind} B={cfg.B} U={cfg.U} {cfg.tracker} K={cfg.K} "
                     f"{1 << cfg.qam_bits}-QAM SNR={cfg.snr_db}dB, {cfg.n_sc} subcarriers x "
                     f"{cfg.S} vectors sharing H" + (", correlated H" if cfg.corr else ""),
         "B": cfg.B, "U": cfg.U, "S": cfg.S, "K": cfg.K,
         "tracker": cfg.tracker, "qam_bits": cfg.qam_bits, "snr_db": cfg.snr_db,
         "parallelism": (f"subcarrier shards: {cfg.n_sc} subcarriers split over {world} GPU(s)"
                         if strong else f"subcarrier shards: {cfg.n_sc} subcarriers per GPU")}
    if strong:
        d["n_sc_total"] = cfg.n_sc
        d["vectors_per_step"] = cfg.vectors
    else:
        d["n_sc_per_gpu"] = cfg.n_sc
        d["vectors_per_step_per_gpu"] = cfg.vectors
    if frames is not None:
        d["l2"] = (f"inputs larger than L2: steps rotate over {frames['n']} frame(s), "
                   f"{frames['bytes'] / 1e6:.0f} MB of H+Y per GPU in total (> 126 MB L2)")
    return d


NVLINK_GBS = 770.0  # measured peer copy per direction (B200_PROFILING.md)


def sharded_gather_pass(args, ctx, cfg_all, cfg, frame, rank, world, local_rank, barrier,
                        max_over_ranks):
    """cfg5 at N > 1, the whole job as north_star states it: each rank runs its
    shard of subcarriers in chunks through the product C ABI and chunk c's
    LLRs, precoded vectors q and s, gains and status bytes go to rank 0 by
    cgm_gatherv (NCCL over NVLink) on a second stream while chunk c + 1 is
    computed (parallel.ShardedPipeline).  Timed with CUDA events, max over
    ranks; the gather term of the path roofline is the bytes that must reach
    rank 0 over its NVLink at the measured per-direction bandwidth."""
    import torch
    import torch.distributed as dist

    from paper_1404_0424_b200 import Context
    from paper_1404_0424_b200.parallel import (Comm, NcclTransport, ShardedPipeline,
                                               detect_precode_outputs)

    uid = [Comm.unique_id() if rank == 0 else None]
    if dist.is_initialized():
        dist.broadcast_object_list(uid, src=0)
    comm_ctx = Context(local_rank)
    comm = Comm(comm_ctx, world, rank, uid[0])
    spec = detect_precode_outputs(cfg_all)
    n_chunks = args.gather_chunks
    pipe = ShardedPipeline(cfg_all.n_sc, rank, world, spec, NcclTransport(comm),
                           n_chunks=n_chunks, device=torch.device("cuda", local_rank))
    H, Y, T = frame
    S, U = cfg.S, cfg.U
    dev = H.device
    scratch = {"xhat": torch.empty((cfg.n_sc, S, U), dtype=torch.complex64, device=dev),
               "mu": torch.empty((cfg.n_sc, S, U), dtype=torch.float32, device=dev),
               "rho": torch.empty((cfg.n_sc, S, U), dtype=torch.float32, device=dev)}

    def compute(a, b, views):
        o = {k: v[a:b] for k, v in scratch.items()}
        o.update(views)
        ctx.detect_precode_cg(H[a:b], Y[a:b], cfg.rho_u, cfg.n0, cfg.es, cfg.qam_bits, cfg.K,
                              cfg.tracker, T[a:b], cfg.rho_d, cfg.K, out=o)

    def timed(gather, reps):
        for _ in range(2):
            pipe.run(compute, gather=gather)
        torch.cuda.synchronize()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        st = torch.cuda.current_stream(dev)
        e0.record(st)
        for _ in range(reps):
            pipe.run(compute, gather=gather)
        e1.record(st)
        torch.cuda.synchronize()
        return max_over_ranks(e0.elapsed_time(e1) / reps)

    reps = max(3, min(args.steps, 20))
    ms_compute = timed(False, reps)
    ms_total = timed(True, reps)
    per_sc = sum(math.prod(s) * torch.empty((), dtype=d).element_size() for s, d in spec.values())
    lo, hi = pipe.lo, pipe.hi
    to_root = (cfg_all.n_sc - (hi - lo if rank == 0 else 0)) * per_sc
    if rank != 0:
        to_root = 0
    if dist.is_initialized():
        t = torch.tensor([float(to_root)], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        to_root = float(t.item())
    comm.close()
    gather_floor_ms = to_root / (NVLINK_GBS * 1e9) * 1e3
    return {"what": ("chunked sharded job: LLRs, precoded vectors q and s, gains and status bytes "
                     "of every rank to rank 0 by cgm_gatherv (NCCL over NVLink) on a second "
                     "stream, overlapped with the next chunk's kernels"),
            "outputs": sorted(spec), "chunks_per_rank": n_chunks,
            "ms_compute_only": ms_compute, "ms_with_gather": ms_total,
            "value_with_gather": cfg_all.vectors / (ms_total / 1e3),
            "bytes_to_root": to_root,
            "roofline": {"term": "bytes to rank 0 / measured NVLink peer bandwidth per direction",
                         "nvlink_gbs": NVLINK_GBS, "gather_floor_ms": gather_floor_ms,
                         "frac": gather_floor_ms / ms_total}}


def ours_arm(args, rank, world, local_rank):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1404_0424_b200 import Context, get_config

    from paper_1404_0424_b200.parallel import shard_range

    cfg_all = get_config(args.config)
    # cfg5 (the BASELINE 1/2/4/8-GPU metric): its 65,536 subcarriers are split
    # over the ranks (strong scaling); the small configs give every rank a
    # whole batch of its own subcarriers (weak scaling)
    strong = cfg_all.name == "cfg5"
    fps = 1
    if strong:
        sc_lo, sc_hi = shard_range(cfg_all.n_sc, rank, world)
        cfg = cfg_all.scaled(sc_hi - sc_lo)
    else:
        # small configs: a step is a stream of frames in one call (SURVEY 7,
        # hard part 2) -- by default enough frames for ~0.5 M vectors per step
        frame_in = cfg_all.n_sc * (cfg_all.B * cfg_all.U + cfg_all.S * cfg_all.B) * 8
        fps = args.frames_per_step or max(1, int(1e9 // frame_in))  # ~1 GB of H + Y per step
        cfg = cfg_all.scaled(cfg_all.n_sc * fps)
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    ctx = Context(local_rank)
    stream = torch.cuda.current_stream(dev)
    # ---------------------------------------------------------------- frames
    frame_bytes = cfg.n_sc * (cfg.B * cfg.U + cfg.S * cfg.B) * 8
    # rotate over distinct frames so no step re-reads L2-resident inputs
    n_frames = 1 if frame_bytes > 2 * 126e6 else max(3, int(np.ceil(3 * 126e6 / frame_bytes)))
    frames = []
    rs = cfg.rsqrt()
    rs = None if rs is None else torch.tensor(rs)
    for f in range(n_frames):
        sc0 = sc_lo if strong else (rank * n_frames + f) * cfg.n_sc
        if cfg.kind == "downlink":
            Hd, T = ctx.generate_downlink(cfg.B, cfg.U, cfg.n_sc, cfg.S, cfg.seed, cfg.qam_bits, sc0=sc0)
            frames.append((Hd, T))
        else:
            H, Y = ctx.generate_uplink(cfg.B, cfg.U, cfg.n_sc, cfg.S, cfg.seed, cfg.qam_bits, cfg.n0,
                                       sc0=sc0, rsqrt=rs)
            T = (ctx.generate_symbols(cfg.U, cfg.n_sc, cfg.S, cfg.seed, cfg.qam_bits, sc0=sc0)
                 if cfg.kind == "both" else None)
            frames.append((H, Y, T))
    torch.cuda.synchronize()
    out = {}

    def step(i):
        fr = frames[i % n_frames]
        if cfg.kind == "downlink":
            ctx.precode_cg(fr[0], fr[1], cfg.rho_d, cfg.K, out=out)
        elif cfg.kind == "both":
            ctx.detect_precode_cg(fr[0], fr[1], cfg.rho_u, cfg.n0, cfg.es, cfg.qam_bits, cfg.K,
                                  cfg.tracker, fr[2], cfg.rho_d, cfg.K, out=out)
        else:
            ctx.detect_cg(fr[0], fr[1], cfg.rho_u, cfg.n0, cfg.es, cfg.qam_bits, cfg.K,
                          cfg.tracker, out=out)

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # --------------------------------------------------------- device timing
    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    # one CUDA graph per input frame (the same C-ABI call captured on a side
    # stream): the timed steps replay them, so small configs are not bound
    # by the host submitting ~30 us of Python + C-ABI work per call
    graphs, graph_note = None, "off (--no-graphs)"
    if not args.no_graphs:
        try:
            cap = torch.cuda.Stream(dev)
            cap.wait_stream(stream)
            l_cap = ctx.kernel_launches
            with torch.cuda.stream(cap):
                for f in range(n_frames):
                    step(f)
            torch.cuda.synchronize()
            per_step = (ctx.kernel_launches - l_cap) / n_frames
            graphs = []
            for f in range(n_frames):
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=cap):
                    step(f)
                graphs.append(g)
            torch.cuda.synchronize()
            for i in range(args.warmup):
                graphs[i % n_frames].replay()
            torch.cuda.synchronize()
            graph_note = f"on ({n_frames} graphs, one per frame, replayed per step)"
        except Exception as e:  # fall back to direct calls, say why
            graphs, graph_note = None, f"failed: {type(e).__name__}: {str(e)[:120]}"
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    l0 = ctx.kernel_launches
    with ClockSampler(local_rank) as clk:
        evs[0].record(stream)
        for i in range(args.steps):
            if graphs:
                graphs[(args.warmup + i) % n_frames].replay()
            else:
                step(args.warmup + i)
            evs[i + 1].record(stream)
        torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    launches = (int(round(per_step * args.steps)) if graphs else ctx.kernel_launches - l0)
    total_ms = max_over_ranks(evs[0].elapsed_time(evs[-1]))
    # per-kernel durations: the same K steps again with CUDA events around
    # every launch inside the C ABI (on the launch stream); a separate pass
    # so the event records do not perturb the headline timing
    # (chunks serialised on one stream for this pass, so each kernel's window
    # is its own: the timed steps above overlap consecutive chunks' kernels
    # on two streams)
    ctx.set_kernel_policy("serial_chunks")
    ctx.set_profiling(True)
    ctx.kernel_times()
    for i in range(args.steps):
        step(args.warmup + i)
    torch.cuda.synchronize()
    ctx.set_kernel_policy("auto")
    kms, n_pairs = ctx.kernel_times_kinds()
    ch_ms, bs_ms, sv_ms, pq_ms = kms["channel"], kms["moments"], kms["solve"], kms["precoder"]
    ctx.set_profiling(False)
    job_vectors = cfg_all.vectors if strong else world * cfg.vectors  # per step, all ranks (x frames)
    value = job_vectors * args.steps / (total_ms / 1e3)
    # the hot path of one step is one channel + one solve launch per L2 chunk
    kernel_ms = (ch_ms + bs_ms + sv_ms + pq_ms) / args.steps

    # ------------------------------------------------------------ e2e (host)
    def pinned(shape, dtype):
        return torch.empty(shape, dtype=dtype, pin_memory=True).numpy()

    # e2e batches: at most ~512 MB of inputs per call (pinned host memory);
    # the metric is the same vectors/s
    per_sc_in = (cfg.B * cfg.U + cfg.S * cfg.B + (cfg.S * cfg.U if cfg.kind == "both" else 0)) * 8
    e2e_sc = cfg.n_sc if strong else int(min(cfg.n_sc, max(1, 512e6 // per_sc_in)))
    h_frames = []
    for fr in frames[: min(2, n_frames)]:
        hf = []
        for t in fr:
            if t is None:
                hf.append(None)
                continue
            a = pinned((e2e_sc, *tuple(t.shape[1:])), torch.complex64)
            a[...] = t[:e2e_sc].cpu().numpy()
            hf.append(a)
        h_frames.append(hf)
    S, U, B, bits = cfg.S, cfg.U, cfg.B, cfg.qam_bits
    if cfg.kind == "downlink":
        h_out = {"q": pinned((e2e_sc, S, B), torch.complex64),
                 "s": pinned((e2e_sc, S, B), torch.complex64),
                 "gain": pinned((e2e_sc, S), torch.float32),
                 "status": pinned((e2e_sc, S), torch.uint8)}
    else:
        h_out = {"xhat": pinned((e2e_sc, S, U), torch.complex64),
                 "mu": pinned((e2e_sc, S, U), torch.float32),
                 "rho": pinned((e2e_sc, S, U), torch.float32),
                 "llr": pinned((e2e_sc, S, U, bits), torch.float32),
                 "status": pinned((e2e_sc, S), torch.uint8)}
        if cfg.kind == "both":
            h_out.update({"q": pinned((e2e_sc, S, B), torch.complex64),
                          "s": pinned((e2e_sc, S, B), torch.complex64),
                          "gain": pinned((e2e_sc, S), torch.float32),
                          "pstatus": pinned((e2e_sc, S), torch.uint8)})
    h2d = sum(a.nbytes for a in h_frames[0] if a is not None)
    d2h = sum(a.nbytes for a in h_out.values())

    def e2e_step(i):
        fr = h_frames[i % len(h_frames)]
        if cfg.kind == "downlink":
            ctx.precode_cg(fr[0], fr[1], cfg.rho_d, cfg.K, out=h_out)
        elif cfg.kind == "both":
            ctx.detect_precode_cg(fr[0], fr[1], cfg.rho_u, cfg.n0, cfg.es, bits, cfg.K,
                                  cfg.tracker, fr[2], cfg.rho_d, cfg.K, out=h_out)
        else:
            ctx.detect_cg(fr[0], fr[1], cfg.rho_u, cfg.n0, cfg.es, bits, cfg.K, cfg.tracker,
                          out=h_out)

    for i in range(args.warmup):
        e2e_step(i)
    barrier()
    t0 = time.perf_counter()
    for i in range(args.steps):
        e2e_step(i)
    e2e_s = max_over_ranks(time.perf_counter() - t0)
    barrier()
    e2e_vectors = cfg_all.vectors if strong else world * e2e_sc * cfg.S
    e2e_value = e2e_vectors * args.steps / e2e_s
    # the e2e ceiling: this box's pinned copy bandwidth with H2D and D2H at
    # once (the host pipeline overlaps both), measured here
    duplex = pcie_duplex_gbs(dev)
    e2e_roof = {"bound": "pcie", "unit": "GB/s",
                "achieved_h2d": h2d * args.steps / e2e_s / 1e9,
                "achieved_d2h": d2h * args.steps / e2e_s / 1e9,
                "peak_duplex_each": duplex,
                "frac": h2d * args.steps / e2e_s / 1e9 / duplex if duplex else None,
                "note": "peak = pinned 256 MB H2D and D2H copies on two streams at once, measured in this run"}

    # ---------------------------------------------------- gather (N > 1 only)
    gather = None
    if (world > 1 or args.force_gather) and strong and cfg.kind == "both":
        gather = sharded_gather_pass(args, ctx, cfg_all, cfg, frames[0], rank, world, local_rank,
                                     barrier, max_over_ranks)
    elif world > 1 and "llr" in out:
        from paper_1404_0424_b200.parallel import gather_to_root

        llr = out["llr"].reshape(-1)
        gather_to_root(llr, world, rank)  # warm
        torch.cuda.synchronize()
        barrier()
        g0 = torch.cuda.Event(enable_timing=True)
        g1 = torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        reps = 5
        for _ in range(reps):
            gather_to_root(llr, world, rank)
        g1.record(stream)
        torch.cuda.synchronize()
        gms = max_over_ranks(g0.elapsed_time(g1) / reps)
        gather = {"what": "LLRs of every rank's step to rank 0 (NCCL)", "ms": gms,
                  "bytes_to_root": llr.numel() * 4 * (world - 1)}

    # -------------------------------------------------------------- roofline
    # per kernel, from the CUDA-event durations of each launch on its stream:
    #   channel kernel: HBM-bound (Gram + matched filter at ~20 FLOP/B sits
    #     far below the tensor-core ridge), algorithmic bytes = H + y
    #   solve kernel: FP32-core-bound, algorithmic flops = CG + tracker + LLR
    # "roofline" is the kernel with the larger share of the step.
    peaks = load_peaks()
    fp32_peak = 148 * 128 * 2 * peaks["sm_max_mhz"] * 1e6 / 1e12  # TFLOP/s
    fp32_src = (f"derived: 148 SMs x 128 FP32 lanes x 2 x {peaks['sm_max_mhz']:.0f} MHz "
                f"(sm_max_mhz from {peaks['source']}; no measured FP32 figure exists)")
    flops_launch = cfg.flops_per_vector() * cfg.vectors
    bytes_launch = cfg.bytes_per_vector() * cfg.vectors
    ch_s = ch_ms / args.steps / 1e3
    sv_s = sv_ms / args.steps / 1e3
    traffic = read_traffic(cfg.name) or {}

    def kernel_roof(name, flops, nbytes, secs, trf):
        """north_star's roofline for one kernel: the slower of its algorithmic
        FLOPs at the FP32 peak and its algorithmic bytes at the HBM peak
        (SURVEY 8(d)); achieved / frac in that bound's unit."""
        t_fp = flops / (fp32_peak * 1e12)
        t_hbm = nbytes / (peaks["hbm_gbs"] * 1e9)
        hbm = t_hbm >= t_fp
        k = {"kernel": name, "bound": "hbm" if hbm else "fp32",
             "unit": "GB/s" if hbm else "TFLOP/s",
             "peak": peaks["hbm_gbs"] if hbm else fp32_peak,
             "peak_source": f"hbm_gbs of {peaks['source']}" if hbm else fp32_src,
             "algorithmic_flops": flops, "algorithmic_bytes": nbytes,
             "roofline_ms": max(t_fp, t_hbm) * 1e3, "ms": secs * 1e3, "traffic": trf}
        k["achieved"] = ((nbytes / secs / 1e9) if hbm else (flops / secs / 1e12)) if secs > 0 else None
        k["frac"] = k["achieved"] / k["peak"] if k["achieved"] else None
        return k

    # credits: channel = Gram + matched filter over H + Y; moments (exact
    # tracker) = the K - 1 Hermitian basis products once per subcarrier;
    # solve = CG + the moment extraction (O(K U) per vector; the reference's
    # O(U^3) extraction is not performed, so it is not credited) + LLRs
    # (+ precoder), over the outputs (+ t, H re-read)
    k_ch = kernel_roof("channel (Gram + matched filter; tcgen05 for U = 32)",
                       cfg.channel_flops_per_vector() * cfg.vectors,
                       cfg.channel_bytes_per_vector() * cfg.vectors, ch_s, traffic.get("channel"))
    pq_s = pq_ms / args.steps / 1e3
    sep = pq_s > 0  # the precoder runs as its own kernel (detect + precode calls)
    pf = cfg.precoder_flops_per_vector() * cfg.vectors if sep else 0.0
    pb = cfg.precoder_bytes_per_vector() * cfg.vectors if sep else 0.0
    k_sv = kernel_roof("solve (CG + SINR extraction + LLR" + ("" if sep else " [+ precoder]") + ")",
                       cfg.solve_kernel_flops_per_vector() * cfg.vectors - pf,
                       cfg.solve_bytes_per_vector(sep) * cfg.vectors, sv_s, traffic.get("solve"))
    k_pq = (kernel_roof("precoder (q = H_d^H v, gain, s; H re-read)", pf, pb, pq_s,
                        traffic.get("precoder")) if sep else None)
    bs_s = bs_ms / args.steps / 1e3
    k_bs = None
    if bs_s > 0:  # exact tracker: row moments of the Chebyshev basis (cgm_moments.cuh)
        k_bs = kernel_roof("moments (exact tracker: (K-1) Hermitian U x U products + row "
                           "moments per subcarrier)",
                           cfg.basis_flops_per_vector() * cfg.vectors, 0.0, bs_s,
                           traffic.get("moments"))
    shares = ([(sv_s, k_sv), (ch_s, k_ch)] + ([(bs_s, k_bs)] if k_bs else [])
              + ([(pq_s, k_pq)] if k_pq else []))
    dom_s, dom = max(shares, key=lambda x: x[0])
    if ch_s == 0 and sv_s > 0:
        # one fused kernel does the whole path (U <= 16 precoder,
        # cgm_precode_small.cuh): its roofline is the path's, HBM or FP32
        # whichever bounds the config
        t_hbm = bytes_launch / (peaks["hbm_gbs"] * 1e9)
        t_fp = flops_launch / (fp32_peak * 1e12)
        hbm = t_hbm >= t_fp
        dom = {"kernel": "fused (Gram + CG + precoder / detector in one kernel)",
               "bound": "hbm" if hbm else "fp32", "unit": "GB/s" if hbm else "TFLOP/s",
               "peak": peaks["hbm_gbs"] if hbm else fp32_peak,
               "peak_source": f"hbm_gbs of {peaks['source']}" if hbm else fp32_src,
               "algorithmic_bytes": bytes_launch, "algorithmic_flops": flops_launch,
               "ms": sv_s * 1e3, "traffic": traffic.get("fused")}
        dom["achieved"] = (bytes_launch / sv_s / 1e9) if hbm else (flops_launch / sv_s / 1e12)
        dom["frac"] = dom["achieved"] / dom["peak"]
        k_sv = dom
        dom_s = sv_s
        k_ch = {"kernel": "(fused into the single kernel)", "ms": 0.0, "frac": None}
    roof = {"bound": dom["bound"], "achieved": dom["achieved"], "peak": dom["peak"],
            "unit": dom["unit"], "frac": dom["frac"], "traffic": dom["traffic"],
            "peak_source": dom["peak_source"], "kernel": dom["kernel"],
            "share_of_step": dom_s / max(ch_s + bs_s + sv_s + pq_s, 1e-12),
            "kernels": {"channel": k_ch, "solve": k_sv, **({"moments": k_bs} if k_bs else {}),
                        **({"precoder": k_pq} if k_pq else {})},
            "pair": {"kernel_ms": kernel_ms, "launch_pairs_per_step": n_pairs / args.steps,
                     "algorithmic_flops": flops_launch, "algorithmic_bytes": bytes_launch,
                     "tflops": flops_launch / (kernel_ms / 1e3) / 1e12,
                     "hbm_gbs": bytes_launch / (kernel_ms / 1e3) / 1e9}}

    # path roofline, SURVEY 8(d)'s formula for the whole step: time =
    # max(F / P_FP32, Bytes / BW_HBM) over the reference algorithm's counts
    # (the exact tracker's U^3 recursion counted per VECTOR as the reference
    # runs it, although the kernels here need it once per subcarrier; so
    # frac can exceed 1 when the restructured algorithm beats that bound)
    step_s = total_ms / args.steps / 1e3
    t_fp = flops_launch / (fp32_peak * 1e12)
    t_hbm = bytes_launch / (peaks["hbm_gbs"] * 1e9)
    roof["path"] = {"formula": "SURVEY 8(d): max(F/P_FP32, Bytes/BW_HBM), reference-algorithm counts",
                    "bound": "hbm" if t_hbm >= t_fp else "fp32",
                    "algorithmic_flops": flops_launch, "algorithmic_bytes": bytes_launch,
                    "roofline_ms": max(t_fp, t_hbm) * 1e3, "ms": step_s * 1e3,
                    "frac": max(t_fp, t_hbm) / step_s,
                    "tflops": flops_launch / step_s / 1e12,
                    "hbm_gbs": bytes_launch / step_s / 1e9}

    # ----------------------------------------------------------- CPU baseline
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            r = cpu_reference(cfg.name)
            cpu = {"value": r["value"], "unit": UNIT, "cores": r["cores"], "kind": r["kind"],
                   "sample": r["sample"]}
        except Exception as e:  # reported, not fatal
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"failed: {e}"[:300]}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "strong" if strong else "weak", "vs_baseline": None, "impl": "ours",
            "dtype": "complex64",
            "data": "synthetic (seeded device generator, reference Rng streams)",
            "config": {**workload_config(cfg_all, {"n": n_frames, "bytes": n_frames * frame_bytes},
                                         world=world),
                       "cuda_graphs": graph_note,
                       "numerics": ("complex64 / FP32 throughout; the U = 32 Gram and matched "
                                    "filter on tcgen05 tensor cores as a bf16 x 3 split (six "
                                    "products, two TMEM accumulators, FP32-level accuracy) -- not "
                                    "north_star's 3xTF32: kind::tf32 with MN-major operands "
                                    "returned zeros on this B200, and fp16 x 2 missed the "
                                    "contract on cfg5 (DESIGN s4, s12); exact-tracker moment "
                                    "table FP32 up to K = 6, FP64 beyond; contract "
                                    "|d| <= 1e-4 + 1e-3 |ref| against the FP64 reference"),
                       **({} if strong else {"frames_per_step": fps,
                                             "vectors_per_step_per_gpu": cfg.vectors})},
            "llr_gbit_s": value * cfg.U * cfg.qam_bits / 1e9 if cfg.kind != "downlink" else None,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "vectors_per_call_per_gpu": e2e_sc * cfg.S,
                    "roofline": e2e_roof},
            "gpu_launches": launches,
            "roofline": roof,
            "cpu_baseline": cpu,
            "clocks": clk.summary(),
        }
        if gather:
            line["gather"] = gather
        print(json.dumps(line), flush=True)


def pcie_duplex_gbs(dev, nbytes=256 << 20, reps=4):
    """Pinned H2D and D2H copies of nbytes at once on two streams -> GB/s per
    direction (the slower of the two)."""
    import torch
    h_in = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    h_out = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    d_a = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    d_b = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    best = None
    for it in range(reps + 1):
        torch.cuda.synchronize(dev)
        e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        with torch.cuda.stream(s1):
            e[0].record()
            d_a.copy_(h_in, non_blocking=True)
            e[1].record()
        with torch.cuda.stream(s2):
            e[2].record()
            h_out.copy_(d_b, non_blocking=True)
            e[3].record()
        torch.cuda.synchronize(dev)
        ms = max(e[0].elapsed_time(e[1]), e[2].elapsed_time(e[3]))
        if it > 0:
            best = ms if best is None else min(best, ms)
    del h_in, h_out, d_a, d_b
    return nbytes / (best * 1e-3) / 1e9


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg5")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--frames-per-step", type=int, default=0,
                    help="weak-scaling configs: frames of the config per step, in one call "
                         "(default: ~1 GB of H + Y per step)")
    ap.add_argument("--gather-chunks", type=int, default=4,
                    help="N > 1, cfg5: chunks per rank of the overlapped output gather")
    ap.add_argument("--force-gather", action="store_true",
                    help="run the chunked gather pass even at one rank (exercises cgm_gatherv)")
    ap.add_argument("--no-graphs", action="store_true",
                    help="time direct C-ABI calls instead of CUDA-graph replays of them")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    dist_on = args.impl == "ours" and (world > 1 or "RANK" in os.environ)
    if dist_on:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        if args.impl == "reference":
            reference_arm(args, rank, world)
        else:
            ours_arm(args, rank, world, local_rank)
    finally:
        if dist_on:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    main()
