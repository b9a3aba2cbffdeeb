#!/usr/bin/env python
"""Benchmark: 3-D registrations/s on 64x128x128 fp32 pairs (BASELINE.json metric).

Workload (config["workload"]): config-3 phantoms -- the config-2 cardiac-shaped pair
(nested-ellipsoid ventricle, Rician noise, radial contraction + smooth displacement)
with seeds 1000 + i -- registered with the config-2 solver (SSD data term, n = 2,
lambda 0.1, theta (rho) 1.0, 7 composed velocity fields, 10 ADMM x 5 Nesterov = 50
accelerated iterations per field, levels = 1).  A step registers `--pairs-per-gpu`
(default 256: on one GPU exactly config 3's 256 pairs; weak scaling, so N GPUs register
256 N pairs).  Pairs per device launch follow the library's policy (`--chunk` overrides):
device-resident batches run as one launch chunk of up to 256 pairs (long persistent
x-pass tile ranges: 115.1 vs 112.9 registrations/s for 2 x 64 at 128 pairs), host-buffer
batches as 64-pair chunks so one chunk's copies overlap the next chunk's registration.

  value : registrations/s over all ranks, inputs resident in HBM before the timed
          region (dreg_cuda_register_batch_device), L2 flushed between steps.
  e2e   : same metric through the host-buffer C ABI (dreg_cuda_register_batch):
          H2D of both volumes and D2H of phi (AoS) + warped image inside the timed region.
  roofline: the dominant kernel (fused x-pass) timed with CUDA events on its stream,
          algorithmic bytes / time vs MEASURED_PEAKS.json hbm_gbs.
  cpu_baseline: the unmodified reference (oracle/_ref) on this box's host cores.

`--impl reference` times the reference CPU implementation alone (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SHAPE = (64, 128, 128)  # numpy (z, y, x) of "64x128x128" -> Dims3{128,128,64}
METRIC = "3D registrations/sec (64x128x128 fp32)"
UNIT = "registrations/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", type=int, default=3, choices=[1, 2, 3, 4, 5],
                    help="BASELINE config (3 = the metric's batched workload; 1/2/4/5 single-pair lines)")
    ap.add_argument("--dropin-pairs", type=int, default=16,
                    help="pairs timed one per call through dreg_cuda_register_pair (pageable host buffers)")
    ap.add_argument("--pairs", type=int, default=None,
                    help="pairs per step over ALL ranks (config 3: 256, split 256/N per GPU: strong scaling)")
    ap.add_argument("--weak", action="store_true",
                    help="weak scaling: --pairs per GPU instead of in total (distinct seeds on every rank)")
    ap.add_argument("--dry-run", action="store_true",
                    help="CPU check of the launcher: N gloo ranks deal the seeds and gather fake records")
    ap.add_argument("--allow-env", action="store_true",
                    help="allow DREG_* experiment variables (they are echoed in the line either way)")
    ap.add_argument("--order", type=int, default=2)
    ap.add_argument("--chunk", type=int, default=0,
                    help="pairs per device launch (0 = library auto: up to 256 device-resident, 64 from host buffers)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-threads", type=int, default=0)
    return ap.parse_args()


def reg_cfg(order):
    from paper_2109_12688_b200 import synth

    return synth.config_cfg("config3", order=order)


# ---- clocks -------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "200",
                 "-i", str(self.index)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[1]))
                mx.append(float(parts[2]))
            except ValueError:
                continue
            for n, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {
            "sm_mhz": statistics.median(sm) if sm else None,
            "sm_max_mhz": max(mx) if mx else None,
            "reasons": sorted(reasons),
            "samples": len(sm),
        }


# ---- CPU reference --------------------------------------------------------------------
def reference_cpu_lib():
    """(library kind, FFT label) of the reference build used for CPU timing: the
    unmodified reference objects over MKL DFTI when that build loads (a production FFT
    like the FFTW the reference links), else over the portable parity FFT shim."""
    from oracle.oracle import available

    if available("reference_mkl") and os.environ.get("DREG_REF_FFT", "mkl") == "mkl":
        return "reference_mkl", "FFTW3 API over MKL DFTI (libtorch_cpu), single-threaded plans"
    return "reference", "FFTW3 API over the portable double FFT shim (~pocketfft speed)"


def cpu_reference_sample(order: int, threads: int, seed0: int = 1000):
    """`threads` concurrent single-threaded reference register_pair calls (the
    reference's public API, the metric's unit: normalise + smooth, up to 7 velocity
    solves of 50 accelerated ADMM iterations, compositions, final warp) on distinct
    config-3 pairs.  Returns (mean seconds per registration, registrations)."""
    from oracle.oracle import CpuLib
    from paper_2109_12688_b200 import synth

    ref = CpuLib(reference_cpu_lib()[0])
    ref.set_threads(1)
    F, M = synth.make_batch(3, seed0, threads, SHAPE)
    cfg = reg_cfg(order)
    errs = []
    per_call = [0.0] * threads

    def work(i):
        try:
            t = time.perf_counter()
            ref.register_pair(F[i], M[i], cfg)
            per_call[i] = time.perf_counter() - t
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    ts = [threading.Thread(target=work, args=(i,)) for i in range(threads)]
    t0 = time.perf_counter()
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    wall = time.perf_counter() - t0
    if errs:
        raise errs[0]
    # steady-state throughput of one registration per core: cores / mean call time
    # (the wall time of the batch would charge the reference for its slowest pair)
    cpu_reference_sample.last_wall = wall
    return sum(per_call) / threads, threads


def run_reference_arm(args, rank, world):
    if rank != 0:
        return
    from oracle.oracle import available

    cores = args.cpu_threads or os.cpu_count() or 1
    if not available("reference"):
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libdreg_ref.so not built"}))
        return
    # one warm-up sample is enough for a CPU arm (page-in, MKL first-use); each step is a
    # full batch of `cores` registrations (~25-30 s), so more would only lengthen the run
    for _ in range(min(args.warmup, 1)):
        cpu_reference_sample(args.order, cores)
    times, walls = [], []
    for _ in range(args.steps):
        dt, _ = cpu_reference_sample(args.order, cores)
        times.append(dt)
        walls.append(cpu_reference_sample.last_wall)
    t = sum(times) / len(times)
    value = cores / t
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": value,
        "unit": UNIT,
        "n_gpus": args.gpus,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": 1000.0 * sum(walls) / len(walls),
        "mean_ms_per_registration": t * 1000.0,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (seeded config-3 phantoms)",
        "config": {"workload": "config3 pairs (64x128x128), config-2 solver n=%d, 7 fields x 50 iterations" % args.order,
                   "impl_detail": "unmodified reference core (oracle/_ref), one thread per pair; FFT: "
                                  + reference_cpu_lib()[1]},
        "cpu_baseline": {
            "value": value,
            "unit": UNIT,
            "cores": cores,
            "kind": "reference",
            "sample": f"per step: {cores} concurrent single-threaded reference register_pair calls on distinct "
                      f"config-3 pairs (config-2 solver, up to 7 fields x 50 iterations); registrations/s = "
                      f"{cores} / mean per-call seconds; FFT: " + reference_cpu_lib()[1],
        },
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---- our arm ---------------------------------------------------------------------------
def dreg_env() -> dict:
    """DREG_* experiment variables in effect (echoed in the line; refused unless --allow-env)."""
    return {k: v for k, v in sorted(os.environ.items()) if k.startswith("DREG_")}


def workload(args):
    """(config name, numpy shape, synth id, RegCfg, workload text) of the bench line."""
    from paper_2109_12688_b200 import synth

    name = f"config{args.config}"
    c = synth.CONFIGS[name]
    cfg = synth.config_cfg(name, order=args.order if args.config in (2, 3) else None)
    n = cfg.solver.order
    text = {
        "config3": f"config3 pairs at config-2 settings: 64x128x128, SSD, n={n}, lambda 0.1, theta 1.0, "
                   "7 fields x 50 ADMM iterations, levels 1",
    }.get(name, f"{name}: {'x'.join(map(str, c['shape']))}, SSD, n={n}, lambda {c['lambda_']}, "
                f"theta {c['theta']}, {c['warps']} fields x {c['iters']} ADMM iterations, levels 1")
    return name, tuple(c["shape"]), c["synth"], cfg, text, c["seed"]


def run_ours(args, rank, world, local_rank):
    import numpy as np
    import torch

    from paper_2109_12688_b200 import dreg, shard, synth

    dist = world > 1
    if dist:
        import torch.distributed as tdist

    env = dreg_env()
    if env and not args.allow_env:
        raise SystemExit(f"bench.py: DREG_* experiment variables set {env}; unset them or pass --allow-env")
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    name, SHAPE_, synth_id, cfg, wl_text, seed_base = workload(args)
    N = SHAPE_[0] * SHAPE_[1] * SHAPE_[2]
    seeds = shard.rank_seeds(rank, world, args.pairs, args.weak, base=seed_base)
    B = len(seeds)
    if B < 1:
        raise SystemExit(f"bench.py: rank {rank} has no pairs ({args.pairs} pairs over {world} ranks)")
    F = np.zeros((B,) + SHAPE_, np.float32)
    M = np.zeros((B,) + SHAPE_, np.float32)
    synth.make_batch(synth_id, seeds[0], B, SHAPE_, out_fixed=F, out_moving=M)  # contiguous seed block
    tgt = torch.from_numpy(F.reshape(B, N)).to(dev)
    src = torch.from_numpy(M.reshape(B, N)).to(dev)
    phi = torch.empty((B, 3, N), dtype=torch.float32, device=dev)
    warped = torch.empty((B, N), dtype=torch.float32, device=dev)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # > 126 MB L2

    ctx = dreg.Context(local_rank)
    stream = torch.cuda.current_stream(dev)
    ctx.set_stream(stream.cuda_stream)
    ctx.set_batch_chunk(args.chunk)  # 0 = library policy (engine.cu pick_chunk)
    chunk = args.chunk or min(B, 256)
    e2e_chunk = args.chunk or min(B, 64)
    dims = SHAPE_[::-1]

    def step():
        return ctx.register_batch_device(B, tgt.data_ptr(), src.data_ptr(), dims, cfg, phi.data_ptr(),
                                         warped.data_ptr())

    for _ in range(args.warmup):
        res = step()
        flush.zero_()
    torch.cuda.synchronize(dev)
    if dist:
        tdist.barrier()
    clocks = ClockSampler(local_rank)
    clocks.start()
    n0 = ctx.kernel_launches()
    torch.cuda.synchronize(dev)
    if dist:
        tdist.barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    sev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for i in range(args.steps):
        sev[i][0].record(stream)
        res = step()
        sev[i][1].record(stream)
        if i + 1 < args.steps:
            flush.zero_()
    e1.record(stream)
    torch.cuda.synchronize(dev)
    if dist:
        tdist.barrier()
    launches = ctx.kernel_launches() - n0
    step_ms = [round(a0.elapsed_time(a1), 2) for a0, a1 in sev]  # per-step registration time (flush excluded)
    clk = clocks.stop()
    ms_max = shard.max_over_ranks(e0.elapsed_time(e1), dev)
    pairs_all = B * world if args.weak else args.pairs
    value = pairs_all * args.steps / (ms_max / 1000.0)

    # per-pair records (status, velocity_count, solves, folding count, final SAD) -> NCCL all-gather
    recs = []
    for p in range(B):
        js = ctx.jacobian_stats_device(phi[p].data_ptr(), dims)
        r = res[p]
        lg = r.per_level[0]
        recs.append([r.status, r.velocity_count, r.solves, js.nonpositive, lg.mean_sad[lg.warps], js.min_det])
    rec = shard.gather_records(torch.tensor(recs, dtype=torch.float64, device=dev)).cpu().numpy()

    # roofline of the dominant kernel (fused x-pass), CUDA events on the launching stream
    tk = ctx.time_kernels(20, cfg.solver)

    # e2e through the host-buffer C ABI (pinned host memory)
    e2e = None
    if not args.no_e2e:
        hT = torch.from_numpy(F.reshape(B, *SHAPE_)).pin_memory()
        hS = torch.from_numpy(M.reshape(B, *SHAPE_)).pin_memory()
        hP = torch.empty((B, *SHAPE_, 3), dtype=torch.float32).pin_memory()
        hW = torch.empty((B, *SHAPE_), dtype=torch.float32).pin_memory()
        tl, sl = [x.numpy() for x in hT], [x.numpy() for x in hS]
        pl, wl = [x.numpy() for x in hP], [x.numpy() for x in hW]
        import ctypes as C

        from paper_2109_12688_b200 import abi

        Fp = C.POINTER(C.c_float)
        Ta = (Fp * B)(*[C.cast(a.ctypes.data, Fp) for a in tl])
        Sa = (Fp * B)(*[C.cast(a.ctypes.data, Fp) for a in sl])
        Pa = (Fp * B)(*[C.cast(a.ctypes.data, Fp) for a in pl])
        Wa = (Fp * B)(*[C.cast(a.ctypes.data, Fp) for a in wl])
        resb = (abi.PairResult * B)()

        def estep():
            st = ctx.lib.dreg_cuda_register_batch(ctx.h, B, Ta, Sa, abi.dims3(dims), abi.Spacing3(1, 1, 1),
                                                  C.byref(cfg), Pa, Wa, resb)
            ctx._check(st)

        estep()
        flush.zero_()
        torch.cuda.synchronize(dev)
        if dist:
            tdist.barrier()
        t0 = time.perf_counter()
        for i in range(args.steps):
            estep()  # synchronous: returns after the D2H of phi / warped completed
            if i + 1 < args.steps:
                flush.zero_()
                torch.cuda.synchronize(dev)
        et = shard.max_over_ranks(time.perf_counter() - t0, dev)
        e2e = {
            "value": pairs_all * args.steps / et,
            "unit": UNIT,
            "h2d_bytes_per_step": B * 2 * N * 4,
            "d2h_bytes_per_step": B * (3 * N + N) * 4,
            "path": "dreg_cuda_register_batch (host C ABI), pinned host buffers, "
                    f"{e2e_chunk}-pair chunks with copy/compute overlap",
        }

    # the reference user's call: one pair per dreg_cuda_register_pair on pageable host
    # memory (what dreg::register_pair in include/dreg_b200/dreg.hpp does with its
    # std::vector buffers), sequentially -- throughput and single-pair latency
    dropin = None
    if not args.no_e2e and rank == 0:
        k = min(B, args.dropin_pairs)
        tl = [np.ascontiguousarray(F[i]) for i in range(k)]
        sl = [np.ascontiguousarray(M[i]) for i in range(k)]
        ctx.register_pair(tl[0], sl[0], cfg)  # warm-up (single-pair workspace + graph)
        lat = []
        t0 = time.perf_counter()
        for i in range(k):
            t1 = time.perf_counter()
            ctx.register_pair(tl[i], sl[i], cfg)  # fresh numpy (pageable) outputs every call
            lat.append(time.perf_counter() - t1)
        tt = time.perf_counter() - t0
        dropin = {
            "value": k / tt,
            "unit": UNIT,
            "pairs": k,
            "single_pair_latency_ms": {"mean": 1e3 * statistics.mean(lat), "min": 1e3 * min(lat),
                                       "max": 1e3 * max(lat)},
            "h2d_bytes_per_pair": 2 * N * 4,
            "d2h_bytes_per_pair": 4 * N * 4,
            "path": "dreg_cuda_register_pair (= dreg::register_pair), pageable host buffers, one pair per call",
        }

    if rank != 0:
        return
    peaks_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    peak, peak_src = 6650.0, "fallback (B200_PROFILING.md)"
    if os.path.exists(peaks_path):
        with open(peaks_path) as f:
            peak = float(json.load(f)["hbm_gbs"])
        peak_src = "measured (MEASURED_PEAKS.json hbm_gbs)"
    # the two per-iteration kernels; `roofline` describes the one that takes longer
    ss = tk.get("spectral_state", 0)
    kern = {
        "xpass": {
            "what": ("xpass, spectral-state form (x c2r -> v-update -> x r2c; streams grad, diff"
                     + (", v" if ss == 1 else "") + " and the x-spectrum)") if ss else
                    "xpass (fused x c2r + dual/Nesterov + v-update + x r2c)",
            "ms": tk["xpass_ms"], "bytes": tk["xpass_bytes"]},
        "plane": {
            "what": ("plane, spectral-state form (yz FFT -> U_j = V^ + (1-m) Ut_{j-1}, Ut_j, (2m-1) Ut_j / N -> "
                     "yz FFT^-1; 5 half-spectra)") if ss else "plane (yz FFT -> multiplier -> yz FFT^-1)",
            "ms": tk["plane_ms"], "bytes": tk["plane_bytes"]},
    }
    for kv in kern.values():
        kv["GBps"] = kv["bytes"] / (kv["ms"] / 1e3) / 1e9
        kv["frac"] = kv["GBps"] / peak
    dom = max(kern, key=lambda k: kern[k]["ms"])
    achieved = kern[dom]["GBps"]
    traffic, traffic_src = None, None
    prof = os.path.join(ROOT, "profiles", "ss_dram_bytes.json" if ss else "xpass_dram_bytes.json")
    if os.path.exists(prof) and name == "config3":
        with open(prof) as f:
            pj = json.load(f)
        pj = pj.get(dom, pj) if ss else (pj if dom == "xpass" else {})
        if pj.get("pairs"):
            traffic = pj["dram_bytes_per_launch"] / pj["pairs"] * tk["pairs"]
            traffic_src = ("recorded ncu constant, not measured in this run: dram__bytes_read.sum + "
                           f"dram__bytes_write.sum of one {dom} launch ({pj.get('source', 'profiles/')}), "
                           "scaled per pair to this launch")
    it_ms = tk["xpass_ms"] + tk["plane_ms"]
    line = {
        "metric": METRIC if name == "config3" else f"3D registrations/sec ({'x'.join(map(str, SHAPE_))} fp32)",
        "value": value,
        "unit": UNIT,
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_max / args.steps,
        "step_ms_rank0": step_ms,
        "higher_is_better": True,
        "scaling": "weak" if args.weak else "strong",
        "vs_baseline": None,
        "dtype": "f32",
        "data": f"synthetic (seeded {name} phantoms, inputs generated on host then resident in HBM)",
        "config": {
            "workload": wl_text,
            "pairs_per_step": pairs_all,
            "pairs_per_gpu_per_step": B,
            "seeds_rank0": [seeds[0], seeds[-1]],
            "device_chunk_pairs": chunk,
            "e2e_chunk_pairs": e2e_chunk,
            "l2": "flushed between timed steps (512 MiB write); per-step working set >> L2",
            "parallelism": f"pairs sharded over {world} GPU(s) ({'weak' if args.weak else 'strong'}: "
                           f"{B} pairs on rank 0); NCCL all-gather of per-pair records only",
            "dreg_env": env,
        },
        "gpu_launches": int(launches),
        "roofline": {
            "bound": "hbm",
            "kernel": kern[dom]["what"],
            "achieved": achieved,
            "peak": peak,
            "peak_source": peak_src,
            "unit": "GB/s",
            "frac": achieved / peak,
            "traffic": traffic,
            "traffic_source": traffic_src,
            "bytes_per_launch": kern[dom]["bytes"],
            "pairs_per_launch": tk["pairs"],
            "iteration_state": {0: "real-space (w, b fields)", 1: "spectral (U_j, U_{j-1}), change norm on",
                                2: "spectral (U_j, U_{j-1}), no change norm (tol = 0)"}[ss],
            "kernels": kern,
            "xpass_ms": tk["xpass_ms"],
            "plane_ms": tk["plane_ms"],
            "plane_GBps": kern["plane"]["GBps"],
            "iteration_ms_per_pair": it_ms / tk["pairs"],
            "iteration_bytes_per_voxel": (tk["xpass_bytes"] + tk["plane_bytes"]) / tk["pairs"] / N,
            "iteration_frac": (tk["xpass_bytes"] + tk["plane_bytes"]) / (it_ms / 1e3) / 1e9 / peak,
            "precise": bool(tk.get("precise", 0)),
        },
        "clocks": clk,
        "e2e": e2e,
        "e2e_dropin": dropin,
        "pairs": shard.summarize(rec),
    }
    if world == 1 and not args.no_cpu and name == "config3":
        from oracle.oracle import available

        if available("reference"):
            cores = args.cpu_threads or os.cpu_count() or 1
            dt, thr = cpu_reference_sample(args.order, cores)
            line["cpu_baseline"] = {
                "value": thr / dt,
                "unit": UNIT,
                "cores": thr,
                "kind": "reference",
                "sample": f"{thr} concurrent single-threaded reference register_pair calls on distinct config-3 "
                          f"pairs (seeds 1000..{999 + thr}, the GPU step's first pairs), mean {dt:.2f} s per call; "
                          f"registrations/s = {thr} / mean; FFT: " + reference_cpu_lib()[1],
            }
    print(json.dumps(line), flush=True)


# ---- launcher ---------------------------------------------------------------------------
def _free_port() -> int:
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def spawn_ranks(args) -> int:
    """`bench.py --gpus N` outside torchrun: re-launch this script as N ranks (one per
    GPU, torch.distributed.run on 127.0.0.1).  Refuses when the box has fewer GPUs."""
    if not args.dry_run:
        import torch

        have = torch.cuda.device_count()
        if have < args.gpus:
            print(f"bench.py: --gpus {args.gpus} but only {have} CUDA device(s) visible", file=sys.stderr)
            return 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def run_dry(args, rank, world):
    """Launcher check without GPUs: each gloo rank takes its seed block and all-gathers
    fake per-pair records; rank 0 prints the dealing."""
    import torch

    from paper_2109_12688_b200 import shard

    seeds = shard.rank_seeds(rank, world, args.pairs, args.weak)
    rec = torch.tensor([[0, rank, 0, 0, float(s), 1.0] for s in seeds], dtype=torch.float64).reshape(-1, 6)
    allrec = shard.gather_records(rec).numpy()
    t = shard.max_over_ranks(float(rank))
    if rank == 0:
        by_rank = {}
        for r in allrec:
            by_rank.setdefault(int(r[1]), []).append(int(r[4]))
        flat = [s for r in sorted(by_rank) for s in by_rank[r]]
        print(json.dumps({"dry_run": True, "n_gpus": world, "scaling": "weak" if args.weak else "strong",
                          "pairs_total": len(flat), "seeds_by_rank": {r: [v[0], v[-1], len(v)] for r, v in by_rank.items()},
                          "disjoint": len(set(flat)) == len(flat), "max_over_ranks": t}), flush=True)


def main():
    args = parse()
    if args.pairs is None:
        args.pairs = 256 if args.config == 3 else 1
    if "WORLD_SIZE" not in os.environ and args.gpus > 1 and args.impl == "ours":
        sys.exit(spawn_ranks(args))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        return
    if world != args.gpus:
        raise SystemExit(f"bench.py: launched with WORLD_SIZE={world} but --gpus {args.gpus}")
    if args.dry_run:
        import torch.distributed as tdist

        if world > 1:
            tdist.init_process_group("gloo")
        try:
            run_dry(args, rank, world)
        finally:
            if world > 1:
                tdist.destroy_process_group()
        return
    if world > 1:
        import torch
        import torch.distributed as tdist

        torch.cuda.set_device(local_rank)
        tdist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as tdist

            tdist.destroy_process_group()


if __name__ == "__main__":
    main()
