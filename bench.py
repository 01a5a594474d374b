#!/usr/bin/env python
"""Device-timed throughput of the B200 LFA SVD (singular values / second).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 5] [--impl ours|reference]

Workload (BASELINE.json): the metric "singular values/sec (full conv SVD,
device-timed) at 1/2/4/8 B200" is quoted on the config that is sharded
across 1/2/4/8 GPUs -- configs[4], the 5x5 c=256 conv on a 256x256 torus with
singular values AND vectors (16,777,216 values per step).  One step = the
whole hot path on resident fp32 weights: K1 half-grid symbol assembly ->
batched Jacobi SVD (sigma + U + V) -> global descending sort of all n*m*r
values (the reference's s_transform + s_svd window, blocksvd.py:259-277).
Under torchrun each rank solves its contiguous share of the 32,770
conjugate-orbit representatives and the sigma shards are all-gathered (NCCL)
and sorted on every rank; time = max over ranks.  The 17.2 GB field and
34 GB of factors per step dwarf the 126 MB L2, so no flush is needed.

``--impl reference`` times the reference's CPU implementation of the path:
the oracle/ C restatement of its numba kernels (bit-exact with the
reference on this container), on all host cores, on a bounded frequency
sample per step (rank 0 only).
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

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2506_05617_b200 import configs  # noqa: E402


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip the FFT-route / analysis timings")
    ap.add_argument("--cpu-seconds", type=float, default=12.0,
                    help="target CPU work of the cpu_baseline / reference sample")
    ap.add_argument("--no-fp64", action="store_true", help="skip the timed fp64 (1e-10 mode) step")
    ap.add_argument("--launcher-dry-run", action="store_true",
                    help="test hook: spawn the ranks and run the rendezvous / max-over-ranks "
                         "timing on gloo without a GPU (no hot path)")
    return ap.parse_args()


def free_port() -> int:
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def spawn_ranks(args) -> int:
    """`--gpus N` without torchrun: launch N ranks (one process per GPU) with
    torch.distributed.run on 127.0.0.1 and return its exit code.  Fails loudly
    when fewer than N GPUs are visible (the dry-run test hook excepted)."""
    if not args.launcher_dry_run:
        import torch

        have = torch.cuda.device_count()
        if have < args.gpus:
            print(json.dumps({"error": f"--gpus {args.gpus} requested but {have} CUDA device(s) visible"}),
                  flush=True)
            return 1
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={free_port()}",
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.run(cmd).returncode


def launcher_dry_run(args, rank, world):
    """Rendezvous + timing reduction of the N-rank path on gloo (CPU test)."""
    import torch
    import torch.distributed as dist

    dist.init_process_group("gloo")
    try:
        dist.barrier()
        t = torch.tensor([float(rank + 1)], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        if rank == 0:
            print(json.dumps({"metric": "launcher dry run", "n_gpus": world, "ranks_seen": world,
                              "max_over_ranks": float(t.item()), "backend": dist.get_backend()}),
                  flush=True)
    finally:
        dist.destroy_process_group()


def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ---------------------------------------------------------------------------
# algorithmic work
# ---------------------------------------------------------------------------
def half_count(n, m):
    h0 = m // 2 + 1
    return h0 + ((n - 1) // 2) * m + (h0 if (n % 2 == 0 and n > 1) else 0)


def svd_flops(layer, vectors, count=None):
    """Golub-Reinsch counts x4 (complex) per unique block."""
    mr, nc = max(layer.c_out, layer.c_in), min(layer.c_out, layer.c_in)
    per = 4 * (14 * mr * nc * nc + 8 * nc ** 3) if vectors else 4 * (4 * mr * nc * nc - 4 * nc ** 3 / 3)
    return per * (half_count(layer.n, layer.m) if count is None else count)


def asm_bytes(layer, count=None, esz=8):
    cnt = half_count(layer.n, layer.m) if count is None else count
    return cnt * layer.c_out * layer.c_in * esz + layer.c_out * layer.c_in * layer.k * layer.k * 4


def read_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except OSError:
        return {}


# ---------------------------------------------------------------------------
# clocks during the timed region
# ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-i", str(self.gpu), "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.thread.join(timeout=2)
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            for name, flag in zip(names, parts[5:9]):
                if flag.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "samples": len(sm), "reasons": sorted(reasons)}


# ---------------------------------------------------------------------------
# CPU leg: the oracle (C restatement of the reference's numba path)
# ---------------------------------------------------------------------------
def cpu_sample_run(layer, vectors, nfreq, threads, seed=0):
    from oracle import oracle as orc  # checker / CPU baseline only

    w = configs.layer_weights(layer).astype(np.float64)
    F = layer.n * layer.m
    rng = np.random.default_rng(seed)
    fidx = np.sort(rng.choice(F, size=min(nfreq, F), replace=False))
    freqs = orc.grid_frequencies(layer.n, layer.m)[fidx]
    t0 = time.perf_counter()
    blocks = orc.symbol_field(w, freqs=freqs, nthreads=threads)
    if vectors:
        orc.svd_full(blocks, nthreads=threads)
    else:
        orc.svd_values(blocks, nthreads=threads)
    dt = time.perf_counter() - t0
    return len(fidx) * min(layer.c_out, layer.c_in), dt


def cpu_calibrate(wl, threads, target_s):
    layer = max(wl.layers, key=lambda l: l.c_out * l.c_in * min(l.c_out, l.c_in))
    svs, dt = cpu_sample_run(layer, wl.vectors, threads, threads, seed=1)  # one block per thread
    per_round = max(dt, 1e-3)
    rounds = max(1, int(target_s / per_round))
    return layer, threads * rounds


def cpu_baseline(wl, threads, target_s):
    layer, nfreq = cpu_calibrate(wl, threads, target_s)
    svs, dt = cpu_sample_run(layer, wl.vectors, nfreq, threads, seed=2)
    return {
        "value": svs / dt, "unit": "singular values/s", "cores": threads, "kind": "port",
        "sample": (f"{min(nfreq, layer.n * layer.m)} of {layer.n * layer.m} frequencies of layer {layer.c_out}x{layer.c_in} "
                   f"k{layer.k} on {layer.n}x{layer.m} ({'sigma+U+V' if wl.vectors else 'sigma'}), "
                   f"symbol assembly + Jacobi, {dt:.1f} s on {threads} threads of {cpu_model()}; "
                   "rate extrapolates linearly in frequencies (blocks are independent)"),
    }


def run_reference(args, wl, rank):
    if rank != 0:
        return
    threads = host_threads()
    layer, nfreq = cpu_calibrate(wl, threads, max(2.0, args.cpu_seconds / 3))
    for i in range(args.warmup):
        cpu_sample_run(layer, wl.vectors, threads, threads, seed=10 + i)
    tot_sv, tot_t = 0, 0.0
    for i in range(args.steps):
        svs, dt = cpu_sample_run(layer, wl.vectors, nfreq, threads, seed=100 + i)
        tot_sv += svs
        tot_t += dt
    value = tot_sv / tot_t
    line = {
        "metric": "singular values/sec (full conv SVD, device-timed)", "value": value,
        "unit": "singular values/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * tot_t / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded Philox He-normal fp32 weights)", "impl": "reference",
        "config": workload_config(wl, args.gpus),
        "cpu_baseline": {"value": value, "unit": "singular values/s", "cores": threads,
                         "kind": "port",
                         "sample": f"{nfreq} random frequencies per step of the largest layer "
                                   f"({'sigma+U+V' if wl.vectors else 'sigma'}); oracle/ C "
                                   "restatement of the reference's numba kernels (bit-exact "
                                   f"with conv-spectra 0.1.0), {cpu_model()}"},
        "e2e": {"value": value, "unit": "singular values/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def workload_config(wl, ngpu):
    L = wl.layers
    cfg = {"workload": wl.name, "layers": len(L),
           "shapes": sorted({f"{l.c_out}x{l.c_in}k{l.k}@{l.n}x{l.m}" for l in L}),
           "outputs": "sigma+U+V" if wl.vectors else "sigma",
           "singular_values_per_step": wl.sv_count,
           "unique_blocks_per_step": sum(half_count(l.n, l.m) for l in L),
           "l2": "inputs larger than L2 (no flush needed)" if wl.name.startswith("cfg5")
                 else "L2 not flushed between steps",
           "parallelism": f"frequency-shard x{ngpu}" if ngpu > 1 else "1 GPU"}
    return cfg


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def fp64_step(wl, layer, w32, dev):
    """One timed fp64 step (the 1e-10 parity mode, like-for-like with the
    reference's complex128 arithmetic): K1 -> warm-started Jacobi with U, V ->
    sort, in float64, device-timed, no warm-up.  Roofline against the DFMA
    rate measured on this GPU; sampled parity against the reference's
    golden sigma (tests/golden, made by the reference itself)."""
    import torch

    import paper_2506_05617_b200 as cs
    from paper_2506_05617_b200 import engine

    torch.cuda.empty_cache()
    w64 = w32.double()
    tm = engine.Timer(dev)
    res = cs.lfa_device(w64, layer.n, layer.m, "f64", wl.vectors, timer=tm)
    torch.cuda.synchronize(dev)
    total = tm.seconds("t0", "t3")
    svd_s = tm.seconds("t1", "t2")
    info = res.info.cpu().numpy()
    peak = engine.fma_peak_flops("f64", dev.index)
    fl = svd_flops(layer, wl.vectors)
    out = {"value": wl.sv_count / total, "unit": "singular values/s", "ms_per_step": 1e3 * total,
           "svd_ms": 1e3 * svd_s, "sweeps_mean": float(info.mean()), "converged": bool((info > 0).all()),
           "roofline": {"bound": "fp64", "achieved": fl / svd_s / 1e12, "peak": peak / 1e12,
                        "unit": "TFLOP/s", "frac": fl / svd_s / peak,
                        "peak_source": "cs_measure_fma_peak(CS_F64) on this GPU in this run",
                        "algorithmic": "Golub-Reinsch count x4 complex per unique block (SURVEY 8(d))"},
           "what": "one fp64 step, no warm-up (plans cached by the fp32 steps)"}
    gpath = os.path.join(ROOT, "tests", "golden", "golden.npz")
    key = f"{wl.name.split('_')[0]}_l0"
    if os.path.exists(gpath):
        g = np.load(gpath)
        if key + "_sigma" in g.files:
            rep_of, _ = engine.partner_map(layer.n, layer.m)
            sig = res.sigma.cpu().numpy()[rep_of[g[key + "_fidx"]]]
            ref = g[key + "_sigma"]
            err = float((np.abs(sig - ref).max(axis=1) / ref[:, 0]).max())
            out["parity"] = {"frequencies": int(len(ref)), "max_rel_err": err, "bar": 1e-10,
                             "ok": err <= 1e-10,
                             "reference": "tests/golden/golden.npz (the reference's own sigma)"}
    del res
    torch.cuda.empty_cache()
    return out


def run_ours(args, wl, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import paper_2506_05617_b200 as cs
    from paper_2506_05617_b200 import engine
    from paper_2506_05617_b200.distributed import lfa_sharded, shard_ids

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    dt = "f32"
    layers = wl.layers
    w_dev = [torch.from_numpy(configs.layer_weights(l)).to(dev) for l in layers]
    fma_peak = engine.fma_peak_flops("f32", local_rank)
    peaks = read_peaks()

    def step(timers=None):
        if len(layers) > 1 and world == 1:  # cfg4: every layer in one batched call
            tm = timers[0] if timers else None
            return cs.lfa_device_multi([(w, l.n, l.m) for l, w in zip(layers, w_dev)], dt,
                                       wl.vectors, timer=tm)
        outs = []
        for i, (l, w) in enumerate(zip(layers, w_dev)):
            tm = timers[i] if timers else None
            # the solve compute_spectrum runs: values-only calls run the vectors
            # solve (factors dropped) whenever that is the panel/tensor-core kernel,
            # so values_only True/False agree bitwise (CS/pipeline.py:40-42)
            vec = wl.vectors or engine.values_via_vectors(engine.half_grid_count(l.n, l.m),
                                                         l.c_out, l.c_in, dt)
            if world > 1:
                outs.append(lfa_sharded(w, l.n, l.m, dt, vec, timer=tm))
            else:
                outs.append(cs.lfa_device(w, l.n, l.m, dt, vec, timer=tm))
        return outs

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(args.warmup):
        outs = step()
    torch.cuda.synchronize(dev)
    info = torch.cat([o.info for o in outs]).float()
    sweeps_mean = float(info.mean().item())
    ok = bool((info > 0).all().item())

    # timed region
    sampler = ClockSampler(dev.index)
    barrier()
    torch.cuda.synchronize(dev)
    sampler.start()
    time.sleep(0.3)
    stream = torch.cuda.current_stream(dev)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    timers = [[engine.Timer(dev) for _ in layers] for _ in range(args.steps)]
    if len(layers) > 1 and world == 1:
        timers = [[engine.Timer(dev)] for _ in range(args.steps)]
    ev[0].record(stream)
    for s in range(args.steps):
        outs = step(timers[s])
        ev[s + 1].record(stream)
    torch.cuda.synchronize(dev)
    barrier()
    clocks = sampler.stop()
    step_ms = [ev[s].elapsed_time(ev[s + 1]) for s in range(args.steps)]
    total_ms = sum(step_ms)
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    svs = wl.sv_count
    value = svs * args.steps / (total_ms / 1e3)

    # per-phase / per-kernel device times (1 GPU: events inside the step)
    roofline = None
    roofline_k1 = None
    phases = None
    if True:  # per-rank phases; at N > 1 the work below is this rank's share
        k1 = [tm.seconds("t0", "t1") for row in timers for tm in row if "t0" in tm.events]
        sv = [tm.seconds("t1", "t2") for row in timers for tm in row if "t0" in tm.events]
        asm = [tm.seconds("t2", "t3") for row in timers for tm in row if "t0" in tm.events]
        nl = len(layers)
        phases = {"assembly_K1_ms": 1e3 * sum(k1) / args.steps,
                  "svd_ms": 1e3 * sum(sv) / args.steps,
                  "spectrum_sort_ms": 1e3 * sum(asm) / args.steps}
        shares = [(len(shard_ids(l.n, l.m, rank, world)) if world > 1 else None) for l in layers]
        svd_flops_step = sum(svd_flops(l, wl.vectors, c) for l, c in zip(layers, shares))
        svd_s = sum(sv) / args.steps
        achieved = svd_flops_step / svd_s / 1e12
        roofline = {"kernel": "SVD phase summed over its launches: jacobi_tcb_kernel (tensor-core "
                              "blocked Jacobi, warm stages of 256x256+V) / jacobi_panel_kernel (seeds, "
                              "other shapes) + warm-start GEMMs",
                    "bound": "fp32", "achieved": achieved, "peak": fma_peak / 1e12,
                    "unit": "TFLOP/s", "frac": achieved * 1e12 / fma_peak,
                    "traffic": None,
                    "peak_source": "measured on this GPU in this run (cs_measure_fma_peak: "
                                   "dependent-FFMA probe); MEASURED_PEAKS.json holds no FP32 peak",
                    "algorithmic": ("Golub-Reinsch sigma+U+V count x4 complex per unique block (SURVEY 8(d))"
                                    if wl.vectors else
                                    "Golub-Reinsch sigma-only count x4 complex per unique block (SURVEY 8(d))")}
        # DRAM traffic per step from the committed ncu capture of this workload
        # (profiles/r02_traffic_cfg5.json; null for other workloads / N > 1):
        # the SVD phase = warm-start GEMMs + K3 + the seeds' K2 launch
        trf = {}
        tpath = os.path.join(ROOT, "profiles", "r02_traffic_cfg5.json")
        if world == 1 and os.path.exists(tpath):
            tj = json.load(open(tpath))
            if tj.get("workload") == workload_config(wl, world).get("workload"):
                trf = tj["per_step"]
        svd_k = [k for k in ("jacobi_tcb_kernel", "warm_gemm_tc_kernel", "jacobi_panel_kernel") if k in trf]
        if svd_k:
            roofline["traffic"] = sum((trf[k]["dram_read_GB"] + trf[k]["dram_write_GB"]) * 1e9 for k in svd_k)
            roofline["traffic_source"] = ("ncu dram__bytes_read+write per step of " + " + ".join(svd_k) +
                                          ", profiles/r02_traffic_cfg5.json")
        asm_b = sum(asm_bytes(l, c) for l, c in zip(layers, shares))
        hbm = peaks.get("hbm_gbs", 6650.0)
        k1_s = sum(k1) / args.steps
        roofline_k1 = {"kernel": "symbol_rows_kernel (K1 half-grid assembly)", "bound": "hbm",
                       "achieved": asm_b / k1_s / 1e9, "peak": hbm, "unit": "GB/s",
                       "frac": asm_b / k1_s / 1e9 / hbm,
                       "traffic": ((trf["symbol_rows_kernel"]["dram_read_GB"] +
                                    trf["symbol_rows_kernel"]["dram_write_GB"]) * 1e9
                                   if "symbol_rows_kernel" in trf else None),
                       "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "fallback 6650 GB/s"}

    # e2e through the public API: host weights -> compute_spectrum(values_only=False)
    e2e = None
    if args.e2e_steps > 0:
        kernels = [cs.ConvKernel.from_array(configs.layer_weights(l)) for l in layers]
        h2d = sum(k.device_weights("f32").nbytes for k in kernels)
        d2h = 0
        barrier()
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            if len(layers) > 1 and world == 1:  # one batched call for all layers
                res = cs.compute_spectra(kernels, [cs.SpatialDims(l.n, l.m) for l in layers],
                                         values_only=not wl.vectors, device=dev, dtype="f32")
                d2h += sum(r.values.nbytes for r in res)
                continue
            for k, l in zip(kernels, layers):
                dims = cs.SpatialDims(l.n, l.m)
                if world == 1:
                    res = cs.compute_spectrum(k, dims, values_only=not wl.vectors, device=dev,
                                              dtype="f32")
                    vals = res.values
                else:
                    w = torch.from_numpy(k.device_weights("f32")).to(dev)
                    out = lfa_sharded(w, l.n, l.m, dt, wl.vectors)
                    vals = out.values.cpu().numpy()
                d2h += vals.nbytes
        torch.cuda.synchronize(dev)
        barrier()
        el = time.perf_counter() - t0
        te = torch.tensor([el], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        el = float(te.item())
        e2e = {"value": svs * args.e2e_steps / el, "unit": "singular values/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h // args.e2e_steps,
               "api": ("distributed.lfa_sharded (host weights in, sorted values out)" if world > 1
                       else "paper_2506_05617_b200.compute_spectra(kernels, dims, dtype='f32') (one batched call)"
                       if len(layers) > 1 else
                       f"paper_2506_05617_b200.compute_spectrum(kernel, dims, values_only={not wl.vectors}, "
                       "dtype='f32')")}

    # SURVEY 8(f) rows measured next to the hot path (1 GPU, single layer):
    # the FFT route's assembly (the paper's comparison baseline) vs K1, and
    # the device post-processing of the spectrum this step produced
    extras = None
    if world == 1 and len(layers) == 1 and not args.no_extras:
        l, w = layers[0], w_dev[0]
        vals = outs[0].values
        del outs
        torch.cuda.empty_cache()
        tf = engine.Timer(dev)
        for rep in range(2):  # second repetition timed (cuFFT plan warm)
            tf = engine.Timer(dev)
            tf.mark("t0")
            fld = engine.fft_symbol_field(w, l.n, l.m, dt, half=True, timer=tf)
            tf.mark("t1")
            del fld
        k1_ms = phases["assembly_K1_ms"]
        fft_ms = 1e3 * tf.seconds("t0", "t1")
        ta = engine.Timer(dev)
        ta.mark("a0")
        summ = cs.spectral_summary(vals)
        ta.mark("a1")
        w1 = cs.wasserstein1(vals, vals[::2])
        ta.mark("a2")
        extras = {
            "fft_route_assembly_ms": {"transform": 1e3 * tf.seconds("t0", "tf"),
                                      "gather": 1e3 * tf.seconds("tf", "t1"), "total": fft_ms,
                                      "k1_ms": k1_ms, "k1_speedup": fft_ms / k1_ms,
                                      "what": "embed + batched cuFFT C2C (c_out*c_in 2D DFTs) + "
                                              "gather to the same representative blocks as K1"},
            "analysis_ms": {"spectral_summary": 1e3 * ta.seconds("a0", "a1"),
                            "wasserstein1_vs_half": 1e3 * ta.seconds("a1", "a2"),
                            "values": int(vals.numel()), "sigma_max": summ.sigma_max, "w1": w1},
        }

    fp64 = None
    if world == 1 and len(layers) == 1 and not args.no_fp64:
        fp64 = fp64_step(wl, layers[0], w_dev[0], dev)

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        cpu = cpu_baseline(wl, host_threads(), args.cpu_seconds)

    # kernel launches of ours per step: per layer K1 + the SVD stages (cold seeds
    # + one warm-start GEMM and one Jacobi launch per warm stage, or one Jacobi
    # launch when cold) + zero-column completion (vectors); then gather, CUB
    # onesweep radix sort (histogram + exclusive-sum + 4 passes) and widen
    per_step = 0
    for l in (layers if not (len(layers) > 1 and world == 1) else []):
        total = half_count(l.n, l.m)
        ids = np.arange(total) if world == 1 else shard_ids(l.n, l.m, rank, world)
        if (engine.use_warm_start(total, l.c_out, l.c_in, dt, wl.vectors) or
                (not wl.vectors and engine.use_warm_values(total, l.c_out, l.c_in, dt))):
            stages = len(engine.subset_plan(l.n, l.m, ids, "cpu"))
            per_step += 1 + stages + (stages - 1) + 1
        else:
            per_step += 1 + 1 + (1 if wl.vectors else 0)
    if len(layers) > 1 and world == 1:  # K1 + one Jacobi launch per layer, then per-layer sort
        per_step = len(layers) * (1 + 1 + (1 if wl.vectors else 0) + 1 + 6 + 1)
    else:
        per_step += 1 + 6 + 1
    launches = args.steps * per_step

    if rank == 0:
        line = {
            "metric": "singular values/sec (full conv SVD, device-timed)",
            "value": value, "unit": "singular values/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
            "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded Philox He-normal fp32 weights, BASELINE.json configs)",
            "config": workload_config(wl, world),
            "roofline": roofline, "roofline_assembly": roofline_k1,
            "phases": phases, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "clocks": clocks, "sweeps_mean": sweeps_mean, "converged": ok, "extras": extras,
            "fp64": fp64,
            "step_ms": step_ms,
        }
        print(json.dumps(line), flush=True)


def main():
    args = parse()
    launched = "WORLD_SIZE" in os.environ
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    wl = configs.WORKLOADS[args.config]
    if args.impl == "reference":  # rank 0 alone times the CPU reference path
        run_reference(args, wl, rank)
        return
    if not launched and args.gpus > 1:
        sys.exit(spawn_ranks(args))
    if args.launcher_dry_run:
        launcher_dry_run(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_ours(args, wl, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    main()
