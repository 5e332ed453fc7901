#!/usr/bin/env python
"""bench.py — FlashNorm fused norm+linear on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One "step" = one pass of the whole per-token hot path (SURVEY §8(a) rows 8a-3..8a-6:
A staging, RMS in parallel with the tcgen05 contraction, deferred scale + bias
epilogue) over one batch of the N=1 workload, BASELINE config 3 (Llama-3-8B
prefill: 4096 tokens, RMSNorm + FFN gate||up 4096 -> 2x14336, bf16).  The
offline folds (8a-1, 8a-2) run once per weight load; they are timed separately
and reported under "fold".  Inputs are resident in HBM and larger than L2
(W* = 235 MB > 126 MB), so no L2 flush is needed between steps.

N > 1 (torchrun, one process per GPU): W* is column-sharded across ranks with the
activations replicated (BASELINE.json:5); each rank computes its
N/P columns with no data-path collective; value = total FLOPs / max-over-ranks
time ("scaling": "strong", the total problem is fixed).

Rank 0 prints ONE JSON line.  The decode config (BASELINE config 2, HBM GB/s)
and the unfused two-kernel variant are measured in the same run and reported
as sub-objects.  --impl reference times the fp64 CPU oracle (oracle/) on a
bounded sample of the same workload (the tier's reference arm).
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

METRIC = "fused norm+linear TFLOP/s (prefill) and HBM GB/s (decode) vs B200 roofline"
PREFILL = dict(M=4096, K=4096, N=28672)
DECODE_K, DECODE_N = 4096, 6144
FALLBACK_PEAKS = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d, "measured"
    except Exception:
        return FALLBACK_PEAKS, "fallback"


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _free_port():
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def spawn_cmd(argv, gpus, port):
    """The torchrun command bench.py re-executes itself under for `--gpus N` (N > 1) when it was
    started as a plain process: one rank per GPU over NCCL on this node (the driver's contract)."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
            "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *argv]


def spawn_env(env):
    """NCCL init logging stays on (INIT subsystem only) so the rank count is visible in the log."""
    env = dict(env)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    return env


# ------------------------------------------------------------------ clocks sampler

class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled DURING the measurement window."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                self.rows.append(parts)

    def stop(self):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if self.thread is not None:
            self.thread.join(timeout=2)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}

        def num(x):
            try:
                return float(x)
            except ValueError:
                return None
        sm = [num(r[1]) for r in self.rows if num(r[1]) is not None]
        pw = [num(r[3]) for r in self.rows if num(r[3]) is not None]
        load = [s for s, p in zip(sm, pw) if p is not None and p > 250.0] or sm
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(load) if load else None,
                "sm_max_mhz": max(num(r[2]) or 0 for r in self.rows), "reasons": reasons,
                "samples": len(self.rows), "samples_under_load": len(load),
                "power_w_max": max(pw) if pw else None}


# ------------------------------------------------------------------ CPU oracle leg

_ORACLE_W = {}


def _oracle_weights(K, N):
    """Config-3-shaped weights for the CPU oracle leg (same recipe: W ~ N(0,1/K), g ~ U[0.5,1.5])."""
    if (K, N) not in _ORACLE_W:
        from synth import gen_layer
        Wt, g, _, _ = gen_layer(1, N, K, "bf16")
        _ORACLE_W[(K, N)] = (Wt.T.astype("float64"), g)
    return _ORACLE_W[(K, N)]


def oracle_sample_rate(M_rows: int, K: int, N: int, seed: int = 0, min_seconds: float = 10.0, max_rows=None):
    """Time the fp64 oracle (unfused RMSNorm -> linear, oracle/flashnorm_oracle.py) on a bounded
    sample of rows of the workload; returns (TFLOP/s, rows, seconds, threads)."""
    import numpy as np
    from oracle import flashnorm_oracle as O
    from synth import gen_activations
    W, g = _oracle_weights(K, N)
    a = gen_activations(seed, M_rows, K, "normal", "bf16")
    threads = os.cpu_count() or 1
    try:
        from threadpoolctl import threadpool_info
        info = threadpool_info()
        if info:
            threads = max(int(i.get("num_threads", 1)) for i in info)
    except Exception:
        pass
    rows = 0
    t0 = time.perf_counter()
    while True:
        O.norm_linear(a[rows % M_rows: rows % M_rows + 1], W, g, None, None, 1e-5, "rmsnorm")
        rows += 1
        el = time.perf_counter() - t0
        if (max_rows is not None and rows >= max_rows) or (max_rows is None and el >= min_seconds):
            break
    return 2.0 * rows * K * N / el / 1e12, rows, el, threads


def run_reference(args, ws, rank):
    if ws > 1 and rank != 0:
        return
    K, N = PREFILL["K"], PREFILL["N"]
    # each step: a bounded sample of rows of the config-3 workload
    rates, times = [], []
    for i in range(args.warmup + args.steps):
        r, rows, el, thr = oracle_sample_rate(8, K, N, seed=i, min_seconds=0.0, max_rows=4)
        if i >= args.warmup:
            rates.append(r)
            times.append(el)
    value = sum(2.0 * 4 * K * N for _ in rates) / sum(times) / 1e12
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * statistics.mean(times),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "llama3-8b-prefill rmsnorm+ffn gate||up (config 3), 4-row sample per step",
                   "M": PREFILL["M"], "K": K, "N": N},
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": thr, "kind": "oracle",
                         "sample": f"4 of {PREFILL['M']} rows per step, fp64 numpy, full N={N}"},
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU leg

def run_ours(args, ws, rank, local):
    import torch
    import paper_2407_09577_b200 as fn
    from paper_2407_09577_b200 import build as fnbuild
    from synth import device as SD

    if not torch.cuda.is_available():
        raise SystemExit("bench.py: no CUDA device (there is no CPU fallback)")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if rank == 0:
        fnbuild.build()
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
        dist.barrier()
    fn.lib()
    peaks, peaks_src = load_peaks()
    M, K, N = PREFILL["M"], PREFILL["K"], PREFILL["N"]
    assert N % (8 * ws) == 0
    Nl = N // ws
    stream = torch.cuda.current_stream(dev)

    def barrier_sync():
        torch.cuda.synchronize(dev)
        if ws > 1:
            import torch.distributed as dist
            dist.barrier()
        torch.cuda.synchronize(dev)

    def max_over_ranks(x):
        if ws == 1:
            return x
        import torch.distributed as dist
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- workload: same seeds on every rank; rank p owns rows [p*Nl, (p+1)*Nl) of W*t
    a = SD.activations(1, M, K, dev, torch.bfloat16)
    Wt_full, g, _, _ = SD.layer(1, N, K, dev, torch.bfloat16)
    Wt = Wt_full[rank * Nl:(rank + 1) * Nl].contiguous()
    del Wt_full
    Ws, cs = fn.fold_weights(Wt, g)
    z = torch.empty((M, Nl), dtype=torch.bfloat16, device=dev)

    clocks = ClockSampler(local if os.environ.get("CUDA_VISIBLE_DEVICES") is None else
                          int(os.environ["CUDA_VISIBLE_DEVICES"].split(",")[local]))
    clocks.start()
    time.sleep(0.3)

    # ---- prefill: the headline (device-resident inputs)
    for _ in range(args.warmup):
        fn.linear(a, Ws, cs, eps=1e-5, out=z)
    barrier_sync()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    fn.reset_launch_count()
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    t_start.record(stream)
    for i in range(args.steps):
        ev[i][0].record(stream)
        fn.linear(a, Ws, cs, eps=1e-5, out=z)
        ev[i][1].record(stream)
    t_end.record(stream)
    launches = fn.launch_count()
    barrier_sync()
    total_ms = max_over_ranks(t_start.elapsed_time(t_end))
    kern_ms = max_over_ranks(statistics.mean(s.elapsed_time(e) for s, e in ev))  # slowest rank's shard
    flops_rank = 2.0 * M * K * Nl
    value = flops_rank * ws * args.steps / (total_ms * 1e-3) / 1e12
    achieved = flops_rank / (kern_ms * 1e-3) / 1e12
    peak_tf = peaks.get("bf16_tflops", FALLBACK_PEAKS["bf16_tflops"])
    # the kernel flashnorm_linear dispatches for this shape (include/flashnorm.h fn_path)
    kname = "flashnorm_gemm2_kernel" if M > 128 else "flashnorm_gemm_kernel"
    # DRAM bytes per launch of this kernel from the latest committed `ncu --set full` capture
    # (profiles/traffic.json names the capture it came from); not re-measured inside this run
    traffic, traffic_src = None, None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        try:
            tj = json.load(open(tp))
            traffic = tj.get(kname)
            traffic_src = tj.get("source")
        except Exception:
            traffic = None

    extra = {}
    if rank == 0 and ws == 1:
        extra = measure_secondary(args, fn, torch, dev, stream, peaks, a, Ws, cs, g)
    if ws > 1:
        extra["multi_gpu"] = measure_multi_gpu(args, fn, torch, dev, stream, a, Ws, cs, z, ws, rank,
                                               barrier_sync, max_over_ranks)
    extra["config5"] = measure_config5(args, fn, torch, dev, stream, peaks, ws, rank, barrier_sync,
                                       max_over_ranks)

    # ---- e2e: through the C ABI with HOST buffers, copies inside the timed region
    a_host = a.cpu().pin_memory()
    z_host = torch.empty((M, Nl), dtype=torch.bfloat16).pin_memory()
    a_dev = torch.empty_like(a)
    e2e_steps = max(3, min(args.steps, 10))
    for _ in range(2):
        fn.linear_from_host(a_host, Ws, cs, a_dev, z, z_host)
    barrier_sync()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(e2e_steps):
        fn.linear_from_host(a_host, Ws, cs, a_dev, z, z_host)
    e1.record(stream)
    barrier_sync()
    e2e_ms = max_over_ranks(e0.elapsed_time(e1))
    e2e_value = flops_rank * ws * e2e_steps / (e2e_ms * 1e-3) / 1e12
    # the link this path is bound by: bare pinned D2H copies of the same z (PCIe), in the same 8
    # row chunks the pipeline uses (one 235 MB copy_ ran at 33-56 GB/s across boxes, chunks steadier)
    zc, zhc = z.chunk(8, 0), z_host.chunk(8, 0)

    def d2h():
        for src, dst in zip(zc, zhc):
            dst.copy_(src, non_blocking=True)
    for _ in range(2):
        d2h()
    torch.cuda.synchronize(dev)
    e0.record(stream)
    for _ in range(e2e_steps):
        d2h()
    e1.record(stream)
    torch.cuda.synchronize(dev)
    d2h_gbs = M * Nl * 2 * e2e_steps / (e0.elapsed_time(e1) * 1e-3) / 1e9
    e2e_link_ms = (M * Nl * 2) / (d2h_gbs * 1e9) * 1e3  # the D2H alone, per step

    clocks.stop()
    if rank != 0:
        return
    cpu = None
    if ws == 1 and not args.no_cpu_baseline:
        r, rows, el, thr = oracle_sample_rate(16, K, N, min_seconds=args.cpu_seconds)
        cpu = {"value": r, "unit": "TFLOP/s", "cores": thr, "kind": "oracle",
               "sample": f"{rows} rows of config 3 (K={K}, N={N}) through the fp64 unfused oracle, {el:.1f} s"}
    line = {
        "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": "llama3-8b-prefill: RMSNorm + FFN gate||up (BASELINE config 3)",
                   "M": M, "K": K, "N": N, "N_per_rank": Nl, "mode": "rmsnorm", "eps": 1e-5,
                   "parallelism": f"column-sharded W* x{ws}" if ws > 1 else "single GPU",
                   "l2": "inputs > L2 (W* 235 MB), no flush"},
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak_tf, "unit": "TFLOP/s",
                     "frac": achieved / peak_tf, "traffic": traffic, "traffic_source": traffic_src,
                     "algorithmic_bytes": (M * K + Nl * K + M * Nl) * 2,
                     "kernel": f"{kname}<MODE_RMS> (tcgen05{' cta_group::2' if M > 128 else ''})",
                     "peak_source": f"{peaks_src} bf16_tflops (burst, cuBLAS)"},
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_value, "unit": "TFLOP/s", "h2d_bytes_per_step": M * K * 2,
                "d2h_bytes_per_step": M * Nl * 2, "steps": e2e_steps,
                "ms_per_step": e2e_ms / e2e_steps, "d2h_link_GB/s": d2h_gbs,
                "frac_of_d2h_link_bound": e2e_link_ms / (e2e_ms / e2e_steps),
                "note": "bound by the PCIe D2H of z: d2h_link_GB/s = bare pinned copies of the same z in 8 row chunks"},
        "gpu_launches": launches,
        "clocks": clocks.summary(),
    }
    line.update(extra)
    print(json.dumps(line), flush=True)


def _events_ms(torch, stream, fnc, steps):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(stream)
    for i in range(steps):
        fnc(i)
    e.record(stream)
    e.synchronize()
    return s.elapsed_time(e) / steps


def measure_multi_gpu(args, fn, torch, dev, stream, a, Ws, cs, z, ws, rank, barrier_sync, max_over_ranks):
    """N > 1 only: how many ranks NCCL sees, and the OPT-IN output gathers timed apart from the
    metric (the shard needs no collective; the gather runs only when asked for).
      * nccl_gather: torch.distributed all_gather_into_tensor (NCCL over NVLink) + the library's
        [P][M][N/P] -> [M][N] permute, after the shard's linear;
      * fused_gather: flashnorm_linear_gather into every rank's symmetric-memory buffer (peer
        stores from the GEMM epilogue) + the device barriers (dist.ColumnParallelFlashNorm).
    Times are device events, max over ranks; each also reports a bit-exact check against the
    NCCL result on this rank."""
    import torch.distributed as dist
    from paper_2407_09577_b200.dist import ColumnParallelFlashNorm
    one = torch.ones(1, device=dev)
    dist.all_reduce(one)
    out = {"world_size": dist.get_world_size(), "gpus_active": int(one.item()), "backend": dist.get_backend()}
    layer = ColumnParallelFlashNorm(Ws, cs, world=ws, rank=rank)
    steps = max(3, min(args.steps, 10))
    try:
        for _ in range(2):
            zg = layer(a, gather=True)
        barrier_sync()
        ms_lin = max_over_ranks(_events_ms(torch, stream, lambda i: fn.linear(a, Ws, cs, eps=1e-5, out=z), steps))
        ms_g = max_over_ranks(_events_ms(torch, stream, lambda i: layer(a, gather=True), steps))
        out["nccl_gather"] = {"linear_ms": ms_lin, "linear_plus_gather_ms": ms_g, "gather_ms": ms_g - ms_lin,
                              "gathered_bytes_per_rank": (ws - 1) * z.numel() * 2}
    except Exception as e:  # reported, never fatal for the metric line
        out["nccl_gather"] = {"error": repr(e)[:300]}
        zg = None
    for key, mc in (("fused_gather", "auto"), ("fused_gather_peer_stores", False)):
        try:
            for _ in range(2):
                layer.forward_fused_gather(a, eps=1e-5, multicast=mc)
            barrier_sync()
            ms_f = max_over_ranks(_events_ms(torch, stream,
                                             lambda i: layer.forward_fused_gather(a, eps=1e-5, multicast=mc), steps))
            zf = layer.forward_fused_gather(a, eps=1e-5, copy=True, multicast=mc)
            barrier_sync()
            same = bool(zg is not None and torch.equal(zf.view(torch.int16), zg.view(torch.int16)))
            out[key] = {"ms": ms_f, "bit_exact_vs_nccl": same, "stores": layer.last_gather}
        except Exception as e:
            out[key] = {"error": repr(e)[:300]}
        if key == "fused_gather" and out[key].get("stores") != "multicast":
            break  # no NVLS mapping: "auto" already measured the peer stores
    return out


def measure_config5(args, fn, torch, dev, stream, peaks, ws, rank, barrier_sync, max_over_ranks):
    """BASELINE config 5 (Llama-3-70B FFN shapes: 8192 tokens, RMSNorm + FFN gate||up 8192 ->
    2 x 28672) with W* column-sharded over the ws ranks: this rank's N/ws columns, activations
    replicated, no collective.  TFLOP/s per rank (slowest rank) and for the whole job."""
    from synth import device as SD
    M, K, N = 8192, 8192, 57344
    Nl = N // ws
    a5 = SD.activations(5, M, K, dev, torch.bfloat16)
    W5, g5, _, _ = SD.layer(5, N, K, dev, torch.bfloat16)
    W5s = fn.fold_weights(W5[rank * Nl:(rank + 1) * Nl].contiguous(), g5)[0]
    del W5
    z5 = torch.empty((M, Nl), dtype=torch.bfloat16, device=dev)
    for _ in range(2):
        fn.linear(a5, W5s, None, eps=1e-5, out=z5)
    barrier_sync()
    steps = 5
    ms = max_over_ranks(_events_ms(torch, stream, lambda i: fn.linear(a5, W5s, None, eps=1e-5, out=z5), steps))
    fl = 2.0 * M * K * Nl
    peak = peaks.get("bf16_tflops", FALLBACK_PEAKS["bf16_tflops"])
    res = {"workload": f"llama3-70b FFN gate||up M={M} K={K} N={N}, column shard N/{ws} = {Nl} per rank",
           "ms_per_step": ms, "TFLOP/s_per_rank": fl / (ms * 1e-3) / 1e12,
           "frac_bf16_peak_per_rank": fl / (ms * 1e-3) / 1e12 / peak,
           "TFLOP/s_job": fl * ws / (ms * 1e-3) / 1e12, "steps": steps}
    del a5, W5s, z5
    torch.cuda.empty_cache()
    return res


def measure_secondary(args, fn, torch, dev, stream, peaks, a, Ws, cs, g):
    """Decode (config 2) HBM GB/s, the unfused two-kernel variant, and the folds."""
    from synth import device as SD
    out = {}
    hbm = peaks.get("hbm_gbs", FALLBACK_PEAKS["hbm_gbs"])

    def timed(fnc, steps, warm=3, graph=False):
        """ms per call.  graph=True: the `steps` calls are captured once into a CUDA graph
        and replayed (launch-bound decode: what a serving loop does), timed with events."""
        for _ in range(warm):
            fnc(0)
        torch.cuda.synchronize(dev)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if not graph:
            s.record(stream)
            for i in range(steps):
                fnc(i)
            e.record(stream)
            torch.cuda.synchronize(dev)
            return s.elapsed_time(e) / steps
        g = torch.cuda.CUDAGraph()
        cs = torch.cuda.Stream(dev)
        with torch.cuda.stream(cs):
            with torch.cuda.graph(g, stream=cs):
                for i in range(steps):
                    fnc(i)
        g.replay()
        torch.cuda.synchronize(dev)
        s.record(stream)
        g.replay()
        e.record(stream)
        torch.cuda.synchronize(dev)
        return s.elapsed_time(e) / steps

    # decode: rotate 8 W* buffers (8 x 50.3 MB = 403 MB >= 3 x the 126 MB L2) so every call
    # streams from HBM.  The decode chain is latency-bound, so let the SM clock recover from the
    # prefill's power cap first
    time.sleep(1.0)
    NB = 8
    Wd = []
    for r in range(NB):
        w, gd, _, _ = SD.layer(100 + r, DECODE_N, DECODE_K, dev, torch.bfloat16)
        Wd.append(fn.fold_weights(w, gd)[0])
        del w
    dec = {}
    for Mdec in (1, 16):
        ad = SD.activations(7, Mdec, DECODE_K, dev, torch.bfloat16)
        zd = torch.empty((Mdec, DECODE_N), dtype=torch.bfloat16, device=dev)
        ms = timed(lambda i: fn.linear(ad, Wd[i % NB], None, eps=1e-5, out=zd), args.secondary_iters, graph=True)
        ms_eager = timed(lambda i: fn.linear(ad, Wd[i % NB], None, eps=1e-5, out=zd), args.secondary_iters)
        byts = DECODE_K * DECODE_N * 2 + Mdec * DECODE_K * 2 + Mdec * DECODE_N * 2
        gbs = byts / (ms * 1e-3) / 1e9
        # unfused: norm kernel + plain GEMV on the original weights (same W stream)
        yd = torch.empty_like(ad)

        def unf(i):
            fn.baseline_norm(ad, g, None, eps=1e-5, out=yd)
            fn.linear(yd, Wd[i % NB], None, mode="none", out=zd)
        ms_u = timed(unf, args.secondary_iters, graph=True)
        gbs_e = byts / (ms_eager * 1e-3) / 1e9
        dec[f"M{Mdec}"] = {"us": ms * 1e3, "GB/s": gbs, "frac_hbm": gbs / hbm, "bytes": byts,
                           "eager_us": ms_eager * 1e3, "eager_GB/s": gbs_e, "eager_frac_hbm": gbs_e / hbm,
                           "unfused_us": ms_u * 1e3, "fusion_gain": ms_u / ms}
    # batched decode (17..128 tokens, K4w): the same W* stream with more tokens per call
    for Mdec in (32, 64):
        ad = SD.activations(7, Mdec, DECODE_K, dev, torch.bfloat16)
        zd = torch.empty((Mdec, DECODE_N), dtype=torch.bfloat16, device=dev)
        ms = timed(lambda i: fn.linear(ad, Wd[i % NB], None, eps=1e-5, out=zd), args.secondary_iters, graph=True)
        byts = DECODE_K * DECODE_N * 2 + Mdec * DECODE_K * 2 + Mdec * DECODE_N * 2
        dec[f"M{Mdec}"] = {"us": ms * 1e3, "GB/s": byts / (ms * 1e-3) / 1e9,
                           "frac_hbm": byts / (ms * 1e-3) / 1e9 / hbm, "bytes": byts,
                           "kernel": "flashnorm_gemv_wide_kernel (batched decode, tokens as the MMA N)"}
    out["decode"] = {"workload": "llama3-8b decode: RMSNorm + QKV 4096->6144 (BASELINE config 2)",
                     "unit": "GB/s", "peak_hbm_gbs": hbm, "l2": f"{NB} rotating W* buffers ({NB * 50.3:.0f} MB >= 3x L2)",
                     "timing": "us/frac_hbm: CUDA graph of back-to-back calls (PDL-chained launches); "
                               "eager_*: the same calls launched one by one from Python; events",
                     "kernel": "flashnorm_gemv_tc_kernel (tcgen05 swap-AB split-K, DSMEM cluster reduction)",
                     **dec}
    del Wd

    # unfused prefill variant: RMSNorm kernel (bf16 y to HBM) then the same GEMM, norm disabled
    M, K, N = a.shape[0], a.shape[1], Ws.shape[0]
    y = torch.empty_like(a)
    z = torch.empty((M, N), dtype=torch.bfloat16, device=dev)
    ms_f = timed(lambda i: fn.linear(a, Ws, cs, eps=1e-5, out=z), 10)

    def unf_p(i):
        fn.baseline_norm(a, g, None, eps=1e-5, out=y)
        fn.linear(y, Ws, None, mode="none", out=z)
    ms_u = timed(unf_p, 10)
    out["unfused_prefill"] = {"fused_ms": ms_f, "unfused_ms": ms_u, "fusion_gain": ms_u / ms_f,
                              "what": "baseline_norm (y=RN(a*r*g)) -> flashnorm_linear(mode=none)"}

    # context only (not part of the library): the vendor GEMM (cuBLAS via torch.matmul) on the same
    # operands, plain bf16 a @ W*^T with no normalization
    ms_cb = timed(lambda i: torch.matmul(a, Ws.t(), out=z), 10)
    out["vendor_gemm_context"] = {"what": "torch.matmul (cuBLAS) a @ W*^T, bf16, no norm — not part of the library",
                                  "ms": ms_cb, "TFLOP/s": 2.0 * M * K * N / (ms_cb * 1e-3) / 1e12}

    # DyT variant of the same shape: tanh pre-pass (K8) into a workspace + the GEMM in mode none,
    # and the in-kernel tanh prologue (MUFU-bound) for comparison
    ws_dyt = torch.zeros(fn.linear_workspace_bytes(M, K, N, "dyt", torch.bfloat16), dtype=torch.uint8, device=dev)
    ms_d = timed(lambda i: fn.linear(a, Ws, cs, mode="dyt", alpha=0.5, out=z, workspace=ws_dyt), 10)
    ms_dp = timed(lambda i: fn.linear(a, Ws, cs, mode="dyt", alpha=0.5, out=z, workspace=None), 5)
    fl = 2.0 * M * K * N
    out["dyt_prefill"] = {"ms": ms_d, "TFLOP/s": fl / (ms_d * 1e-3) / 1e12,
                          "frac_bf16_peak": fl / (ms_d * 1e-3) / 1e12 / peaks.get("bf16_tflops", 1657.2),
                          "prologue_ms": ms_dp, "prologue_TFLOP/s": fl / (ms_dp * 1e-3) / 1e12,
                          "what": "dyt_prepass (tanh once per element) -> GEMM mode none; prologue = tanh in SMEM"}
    del ws_dyt

    # NEXT-1: the same gate||up GEMM with the GLU epilogue (SwiGLU, Fig 3(b)): h [M, F] (half the
    # output bytes) + s [M]; then the down projection F -> K scaled by s at its output
    F = N // 2
    Wgu = fn.fold_glu_weights(Ws[:F], Ws[F:], None)  # W* rows already carry g
    h = torch.empty((M, F), dtype=torch.bfloat16, device=dev)
    sg = torch.empty(M, dtype=torch.float32, device=dev)
    ms_g = timed(lambda i: fn.glu_linear(a, Wgu, eps=1e-5, act="silu", out=h, s_out=sg), 10)
    Wdn, _, _, _ = SD.layer(77, K, F, dev, torch.bfloat16)
    yd = torch.empty((M, K), dtype=torch.bfloat16, device=dev)
    ms_dn = timed(lambda i: fn.linear_scaled(h, Wdn, sg, out=yd), 10)
    fl_g, fl_d = 2.0 * M * K * N, 2.0 * M * F * K
    out["glu_ffn"] = {"workload": "llama3-8b FFN (SwiGLU) at config 3: gate||up 4096->2x14336 with the GLU "
                                  "epilogue, then down 14336->4096 scaled by s (Figs 3(b))",
                      "gate_up_ms": ms_g, "gate_up_TFLOP/s": fl_g / (ms_g * 1e-3) / 1e12,
                      "gate_up_frac_bf16_peak": fl_g / (ms_g * 1e-3) / 1e12 / peaks.get("bf16_tflops", 1657.2),
                      "down_ms": ms_dn, "down_TFLOP/s": fl_d / (ms_dn * 1e-3) / 1e12,
                      "ffn_ms": ms_g + ms_dn, "ffn_TFLOP/s": (fl_g + fl_d) / ((ms_g + ms_dn) * 1e-3) / 1e12}
    del Wgu, h, Wdn, yd

    # NEXT-4: exact LayerNorm deferred past the contraction (mean via u = 1^T W*, reading c29) at the
    # config-3 shape (same CTA-pair kernel as the headline) and at config 4 (2048 x 4096 -> 4096)
    u3 = fn.fold_colsum(Ws)
    ms_ln = timed(lambda i: fn.layernorm_linear(a, Ws, u3, cs, eps=1e-5, out=z), 10)
    a4 = SD.activations(9, 2048, 4096, dev, torch.bfloat16)
    W4, g4, _, _ = SD.layer(9, 4096, 4096, dev, torch.bfloat16)
    W4s, c4s = fn.fold_weights(W4, g4)
    u4 = fn.fold_colsum(W4s)
    z4 = torch.empty((2048, 4096), dtype=torch.bfloat16, device=dev)
    # ~45 us kernels: a CUDA graph of back-to-back calls, or the Python wrapper's per-call cost
    # (not the kernel) is what gets timed
    ms_ln4 = timed(lambda i: fn.layernorm_linear(a4, W4s, u4, c4s, eps=1e-5, out=z4), 20, graph=True)
    ms_rms4 = timed(lambda i: fn.linear(a4, W4s, c4s, eps=1e-5, out=z4), 20, graph=True)
    ms_cs = timed(lambda i: fn.fold_colsum(Ws, out=u3), 10)
    fl4 = 2.0 * 2048 * 4096 * 4096
    out["layernorm_exact"] = {
        "what": "flashnorm_layernorm_linear: z = (a W* - mu u) rsqrt(var + eps) + c*, mu/var beside the MMA",
        "config3_ms": ms_ln, "config3_TFLOP/s": fl / (ms_ln * 1e-3) / 1e12,
        "config3_frac_bf16_peak": fl / (ms_ln * 1e-3) / 1e12 / peaks.get("bf16_tflops", 1657.2),
        "config4_ms": ms_ln4, "config4_TFLOP/s": fl4 / (ms_ln4 * 1e-3) / 1e12,
        "config4_rmsnorm_ms": ms_rms4,
        "fold_colsum_us": ms_cs * 1e3, "fold_colsum_GB/s": N * K * 2 / (ms_cs * 1e-3) / 1e9}
    del a4, W4, W4s, z4, u3, u4

    # folds (offline, once per weight load): config-3 W (235 MB in + 235 MB out); like the decode
    # section, let the SM clock recover from the GEMMs' power cap first
    Wf, gf, bf_, cf = SD.layer(5, N, K, dev, torch.bfloat16, with_b=True, with_c=True)
    torch.cuda.synchronize(dev)
    time.sleep(1.0)
    Wo = torch.empty_like(Wf)
    co = torch.empty(N, dtype=torch.float32, device=dev)
    ms_fold = timed(lambda i: fn.fold_weights(Wf, gf, bf_, cf, out=Wo, c_out=co), 10)
    fb = 2 * N * K * 2 + 3 * K * 4 + 2 * N * 4
    out["fold"] = {"fold_weights_us": ms_fold * 1e3, "GB/s": fb / (ms_fold * 1e-3) / 1e9,
                   "frac_hbm": fb / (ms_fold * 1e-3) / 1e9 / hbm, "bytes": fb, "shape": [N, K]}
    del Wf, Wo
    # LayerNorm retrofit fold (config 4 V: 4096 x 4096 bf16 + b_prev), CUDA graph over 6 rotating
    # V / V* pairs (6 x 67 MB = 403 MB >= 3 x L2): every call reads V from HBM and writes V* to it
    NV = 6
    Vts, bps, Vss = [], [], []
    for r in range(NV):
        _, Vt, bp = SD.upstream(4 + r, 16, 4096, 4096, dev, torch.bfloat16)
        Vts.append(Vt)
        bps.append(bp)
        Vss.append(torch.empty_like(Vt))
    wsv = torch.zeros(fn.fold_mean_center_workspace_bytes(4096, 4096) // 8 + 2, dtype=torch.float64, device=dev)
    ms_mc = timed(lambda i: fn.fold_mean_center(Vts[i % NV], bps[i % NV], out=Vss[i % NV], workspace=wsv), 24,
                  graph=True)
    vb = 2 * 4096 * 4096 * 2
    out["fold"].update({"fold_mean_center_us": ms_mc * 1e3, "fold_mean_center_GB/s": vb / (ms_mc * 1e-3) / 1e9,
                        "fold_mean_center_frac_hbm": vb / (ms_mc * 1e-3) / 1e9 / hbm,
                        "fold_mean_center_shape": [4096, 4096],
                        "fold_mean_center_l2": f"{NV} rotating V/V* pairs ({NV * 67} MB >= 3x L2), CUDA graph"})
    del Vts, Vss
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--secondary-iters", type=int, default=200,
                    help="calls per decode/unfused timing loop (small values for profiler runs)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    ws, rank, local = dist_env()
    if args.impl == "reference":
        run_reference(args, max(ws, args.gpus) if "WORLD_SIZE" not in os.environ else ws, rank)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # `python bench.py --gpus N` as a plain process: become N ranks (one per GPU) under torchrun
        import torch
        n = torch.cuda.device_count()
        if n < args.gpus:
            raise SystemExit(f"bench.py --gpus {args.gpus}: only {n} CUDA device(s) visible")
        sys.exit(subprocess.call(spawn_cmd(sys.argv[1:], args.gpus, _free_port()), env=spawn_env(os.environ)))
    if ws != args.gpus:
        raise SystemExit(f"bench.py: WORLD_SIZE={ws} but --gpus {args.gpus} (one rank per GPU)")
    run_ours(args, ws, rank, local)
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
