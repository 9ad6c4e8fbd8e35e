"""Benchmark: chunked power attention fwd+bwd, BASELINE.json configs[1]
(p=2, d=e=64, b=4, h=16, t=65536, c=1024, gated, bf16) on B200.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]

One step = power_full forward + backward over the whole synthetic batch
(inputs resident in HBM, each 512 MiB >> the 126 MB L2, so no L2 flush is
needed).  Multi-GPU (--gpus N; bench.py re-launches itself under
torch.distributed.run when started without it): one process per GPU, by
default the sequence-parallel 1M-token config (configs[3], chunk ranges per
rank, carry chain over NCCL point-to-point; strong scaling); --workload cfg2
shards configs[1]'s streams instead (weak scaling, no data-path collective).
Timing: CUDA events on the launching stream, barrier + synchronize on both
sides, max over ranks.

--impl reference times the reference's own CPU algorithm (the numpy oracle
port, oracle/power_oracle.py, which is pinned to the reference by
tests/golden) on the host cores: one process per core, each running a bounded
slice of one (batch, head) stream; tokens/s is extrapolated linearly in t
(the chunked form is linear in t, reference test_acceptance.py:345-354).
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

METRIC = "power-attn fwd+bwd tokens/sec at p=2,d=64,64k ctx; % of BF16 tensor peak"
# BASELINE.json configs, numbered as in SURVEY.md (cfg1 = configs[0], ...)
WORKLOADS = {
    "cfg1": (dict(b=1, h=2, t=1024, d=32, e=32, p=2, chunk=128, gated=True, normalize=False, dtype="f32"),
             "configs[0]: power_full fwd+bwd fp32 p=2 d=32 b=1 h=2 t=1024 chunk=128 gated"),
    "cfg2": (dict(b=4, h=16, t=65536, d=64, e=64, p=2, chunk=1024, gated=True, normalize=False, dtype="bf16"),
             "configs[1]: power_full fwd+bwd bf16 p=2 d=64 b=4 h=16 t=65536 chunk=1024 gated"),
    "cfg3": (dict(b=1, h=16, t=16384, d=32, e=32, p=4, chunk=1024, gated=False, normalize=True, dtype="bf16"),
             "configs[2]: power_full fwd+bwd bf16 p=4 d=32 (D=52360) b=1 h=16 t=16384 chunk=1024 ungated, "
             "normalized"),
    # one 1,048,576-token sequence (b=1, h=16) split over the ranks by chunk range
    # (sequence parallelism, carry chain over NCCL point-to-point)
    "sp1m": (dict(b=1, h=16, t=1048576, d=64, e=64, p=2, chunk=1024, gated=True, normalize=False, dtype="bf16"),
             "configs[3]: sequence-parallel power_full fwd+bwd bf16 p=2 d=64 b=1 h=16 t=1048576 chunk=1024 "
             "gated, chunk ranges split over the ranks"),
}
CFG, WORKLOAD = WORKLOADS["cfg2"]


# --------------------------------------------------------------------------
# algorithmic FLOPs (SURVEY section 8d / BASELINE.md: 2 FLOP per MAC, contractions only)
# --------------------------------------------------------------------------
def flops(cfg, ns=None):
    b, h, t, d, e, p, c = (cfg[k] for k in ("b", "h", "t", "d", "e", "p", "chunk"))
    ns = b * h if ns is None else ns
    D = math.comb(d + p - 1, p)
    n = t // c
    ecols = e + (1 if cfg["normalize"] else 0)
    intra = n * c * (c + 1) // 2 * (d + e)
    update = t * D * ecols
    query = (t - c) * D * ecols
    fwd = 2 * ns * (intra + update + query)
    return dict(fwd=fwd, bwd=2 * fwd, total=3 * fwd, intra=2 * ns * intra, update=2 * ns * update,
                query=2 * ns * query)


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return pk.get("bf16_tflops", 1590.0), pk.get("bf16_tflops_sustained", 1400.0), pk.get("hbm_gbs", 6650.0), "measured"
    except Exception:
        return 1590.0, 1400.0, 6650.0, "fallback"


# --------------------------------------------------------------------------
# clocks sampler (B200_PROFILING.md clocks line)
# --------------------------------------------------------------------------
class Clocks:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def mark(self):
        self.m = len(self.lines)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons, power = [], None, set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        m = getattr(self, "m", 0)
        timed = self.lines[m:] if len(self.lines) > m else self.lines[-2:]
        for ln in timed:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
                power.append(float(f[3]))
            except ValueError:
                continue
            for nm, val in zip(names, f[5:9]):
                if val.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm),
                "power_w_max": max(power) if power else None}


# --------------------------------------------------------------------------
# CPU reference arm / baseline (oracle port of the reference algorithm)
# --------------------------------------------------------------------------
def _cpu_worker(args):
    cfg, t_slice, seed = args
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    import numpy as np
    from threadpoolctl import threadpool_limits

    from oracle import power_oracle as O

    with threadpool_limits(1):
        q, k, v, g = O.generate_inputs(1, t_slice, 1, cfg["d"], cfg["e"], seed=seed, dtype=np.float32,
                                       gating=cfg["gated"])
        dy = np.ones_like(v)
        t0 = time.perf_counter()
        O.chunked_forward(q, k, v, g, cfg["p"], cfg["chunk"], normalize=cfg["normalize"])
        O.chunked_backward(q, k, v, g, cfg["p"], cfg["chunk"], dy, normalize=cfg["normalize"])
        return time.perf_counter() - t0


def cpu_sample(cfg, cores: int, t_slice: int | None = None):
    """One bounded sample of the workload on the host: `cores` processes, each
    fwd+bwd over one (batch, head) stream slice of t_slice tokens.  Returns
    (tokens/s of the b*t metric, seconds, description)."""
    import multiprocessing as mp

    if t_slice is None:
        # 8 chunks (query runs on 7 of 8, the full stream on 63 of 64); p=4 streams
        # cost ~50x more per token, so they get one chunk pair
        t_slice = min(cfg["t"], cfg["chunk"] * (2 if cfg["p"] > 2 else 8))
    n_proc = min(cores, cfg["b"] * cfg["h"]) if t_slice >= cfg["t"] else cores
    ctx = mp.get_context("fork")
    t0 = time.perf_counter()
    with ctx.Pool(n_proc) as pool:
        pool.map(_cpu_worker, [(cfg, t_slice, i) for i in range(n_proc)])
    wall = time.perf_counter() - t0
    stream_tok_s = n_proc * t_slice / wall
    tok_s = stream_tok_s / cfg["h"]  # the metric counts b*t tokens; each token spans h streams
    desc = (f"{n_proc} processes x 1 stream x {t_slice} tokens (p={cfg['p']}, d={cfg['d']}, c={cfg['chunk']}, "
            f"gated={cfg['gated']}, normalize={cfg['normalize']}) fwd+bwd, numpy oracle (port of reference "
            f"chunked.py/gradients.py), 1 BLAS thread each; tokens/s = stream-tokens/s / h (linear in t, "
            f"reference test_acceptance.py:345-354)")
    return tok_s, wall, desc


def pick_workload(args, world: int):
    name = args.workload
    if name == "auto":
        name = "cfg2" if world == 1 else "sp1m"
    return name


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    name = pick_workload(args, world)
    if name == "lm124m":
        print(json.dumps({"impl": "reference", "unavailable": "configs[4] is a model stack; the reference has no "
                          "LM (its CPU path is the attention operator only)"}), flush=True)
        return
    cfg, workload = WORKLOADS[name]
    cores = os.cpu_count() or 1
    for _ in range(args.warmup):
        cpu_sample(cfg, cores, cfg["chunk"])
    vals = []
    t_all = time.perf_counter()
    desc = ""
    for _ in range(args.steps):
        v, wall, desc = cpu_sample(cfg, cores)
        vals.append(v)
    elapsed = time.perf_counter() - t_all
    val = statistics.median(vals)
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": "tokens/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * elapsed / max(args.steps, 1),
        "higher_is_better": True, "scaling": "strong" if name == "sp1m" else "weak", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic (Philox, reference inputs.py distributions)",
        "config": {"workload": workload + " (bounded CPU sample, extrapolated)", **cfg},
        "cpu_baseline": {"value": val, "unit": "tokens/s", "cores": cores, "kind": "port", "sample": desc},
        "e2e": {"value": val, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------
# GPU arm
# --------------------------------------------------------------------------
def scan_bytes(cfg):
    """Algorithmic HBM bytes of the two scans per step, fp16 state
    storage: forward reads S_k and writes A_k; backward reads dA_k and A_k and
    writes the state cotangent."""
    D = math.comb(cfg["d"] + cfg["p"] - 1, cfg["p"])
    n, ns = cfg["t"] // cfg["chunk"], cfg["b"] * cfg["h"]
    cols = cfg["e"] + (1 if cfg["normalize"] else 0)
    unit = n * ns * D * cols * 2
    return {"fwd_discumsum": 2 * unit, "bwd_discumsum": 3 * unit}


def run_gpu(args):
    import torch
    import torch.distributed as dist

    from paper_2507_04239_b200 import _lib, power_full
    from paper_2507_04239_b200.parallel import power_full_sp

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    name = pick_workload(args, world)
    if name == "lm124m":
        return run_lm(args, world, rank, local)
    cfg, workload = WORKLOADS[name]
    sp = name == "sp1m"
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    b, h, t, d, e, c = (cfg[k] for k in ("b", "h", "t", "d", "e", "chunk"))
    if sp:
        t = t // world   # this rank's contiguous token range
    dt = torch.float32 if cfg["dtype"] == "f32" else torch.bfloat16
    g = torch.Generator(device=dev).manual_seed(1234 + rank)
    Q = (torch.rand(b, t, h, d, device=dev, generator=g) * 2 - 1).to(dt).requires_grad_()
    K = (torch.rand(b, t, h, d, device=dev, generator=g) * 2 - 1).to(dt).requires_grad_()
    V = (torch.rand(b, t, h, e, device=dev, generator=g) * 2 - 1).to(dt).requires_grad_()
    LG = None
    if cfg["gated"]:
        LG = torch.log(torch.rand(b, t, h, device=dev, generator=g) * 0.1 + 0.9).requires_grad_()
    dY = (torch.rand(b, t, h, e, device=dev, generator=g) * 2 - 1).to(dt)
    ins = [x for x in (Q, K, V, LG) if x is not None]

    def op(q, k, v, lg):
        if sp:
            return power_full_sp(q, k, v, lg, p=cfg["p"], chunk_size=c, normalize=cfg["normalize"])
        return power_full(q, k, v, lg, p=cfg["p"], chunk_size=c, normalize=cfg["normalize"],
                          check_denominator=False)

    def step():
        y = op(Q, K, V, LG)
        return torch.autograd.grad(y, ins, dY)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # the clock sampler starts before the warm-up (nvidia-smi needs a few hundred ms
    # to produce its first line); only samples taken after the mark -- inside the
    # timed region -- count, or the last warm-up samples if the region was shorter
    # than the sampling interval
    clocks = Clocks(local)
    clocks.start()
    for _ in range(args.warmup):
        step()
    barrier()
    clocks.mark()
    _lib.profile_reset()
    _lib.profile_enable(True)
    n0 = _lib.launch_count()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        step()
    e1.record()
    barrier()
    launches = _lib.launch_count() - n0
    _lib.profile_enable(False)
    stages = _lib.profile_read()
    ck = clocks.stop()
    ms = e0.elapsed_time(e1) / args.steps
    if world > 1:
        tt = torch.tensor([ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    tokens = b * t * world
    value = tokens / (ms / 1000.0)

    # ---- e2e: reference-facing call with HOST buffers (copies timed) ------
    e2e = None
    if not args.no_e2e:
        host_in = [x.detach().cpu().pin_memory() for x in ins] + [dY.cpu().pin_memory()]
        # y and every gradient come back to the host each step
        outs = [torch.empty((b, t, h, e), dtype=dt).pin_memory()] + \
               [torch.empty(x.shape, dtype=x.dtype).pin_memory() for x in ins]
        h2d = sum(x.numel() * x.element_size() for x in host_in)
        d2h = sum(x.numel() * x.element_size() for x in outs)

        # Pipelined like a training loop that prefetches its next batch: the
        # host->device copy of step i+1 and the device->host copy of step i-1
        # run on their own streams while step i computes (every byte still
        # crosses PCIe inside the timed region, every step).
        s_comp = torch.cuda.current_stream(dev)
        s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        dbuf = [[torch.empty(x.shape, dtype=x.dtype, device=dev) for x in host_in] for _ in range(2)]
        ev_in = [torch.cuda.Event() for _ in range(2)]
        ev_free = [torch.cuda.Event() for _ in range(2)]
        ev_done = torch.cuda.Event()
        for ev in ev_free:
            ev.record(s_comp)

        def e2e_step(i):
            bi = i % 2
            with torch.cuda.stream(s_in):
                s_in.wait_event(ev_free[bi])
                for dst, src in zip(dbuf[bi], host_in):
                    dst.copy_(src, non_blocking=True)
                ev_in[bi].record(s_in)
            s_comp.wait_event(ev_in[bi])
            xs = [x.detach().requires_grad_() for x in dbuf[bi][:-1]]
            xs4 = xs + [None] * (4 - len(xs))
            y = op(*xs4)
            gr = torch.autograd.grad(y, xs, dbuf[bi][-1])
            ev_free[bi].record(s_comp)
            ev_done.record(s_comp)
            with torch.cuda.stream(s_out):
                s_out.wait_event(ev_done)
                for o, gx in zip(outs, (y.detach(),) + tuple(gr)):
                    gx.record_stream(s_out)
                    o.copy_(gx, non_blocking=True)

        e2e_step(0)
        torch.cuda.synchronize()
        barrier()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(s_comp)
        # as many pipelined steps as the device-timed region: the first H2D and the
        # last D2H (pipeline fill / drain) are inside the timed region either way
        ne = max(4, args.steps)
        for i in range(ne):
            e2e_step(i)
        s_comp.wait_stream(s_out)
        f1.record(s_comp)
        barrier()
        ems = f0.elapsed_time(f1) / ne
        if world > 1:
            tt = torch.tensor([ems], device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ems = float(tt.item())
        e2e = {"value": tokens / (ems / 1000.0), "unit": "tokens/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": ems,
               "pipeline": "H2D of step i+1 and D2H (y and all gradients) of step i-1 overlap step i"}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    peak, peak_sus, hbm, peak_kind = load_peaks()
    fl = flops(cfg)
    jobs = 1 if sp else world   # the whole-job algorithmic FLOPs
    tflops = jobs * fl["total"] / (ms / 1000.0) / 1e12
    # dominant kernel (largest share of step time) and its roofline
    stage_ms = {k: v[0] / args.steps for k, v in stages.items()}
    stage_n = {k: v[1] / args.steps for k, v in stages.items()}
    roof = None
    if stage_ms:
        dom = max(stage_ms, key=stage_ms.get)
        per = stage_flops(dom, fl)
        if per is not None and sp:
            per /= world   # stage times are per rank; fl is the whole sequence
        if per is not None:
            launch_ms = stage_ms[dom] / max(stage_n[dom], 1)
            achieved = per / max(stage_n[dom], 1) / (launch_ms / 1000.0) / 1e12
            roof = {"kernel": dom, "bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                    "frac": achieved / peak, "traffic": traffic_for(dom),
                    "peak_kind": f"{peak_kind} burst bf16 (cuBLAS, MEASURED_PEAKS.json); sustained {peak_sus}",
                    "frac_of_sustained": achieved / peak_sus, "share_of_step": stage_ms[dom] / ms}
    scans = {}
    for st_name, nbytes in scan_bytes(cfg).items():
        if st_name in stage_ms and stage_ms[st_name] > 0:
            per_rank = nbytes / (world if sp else 1)
            gbs = per_rank / (stage_ms[st_name] / 1000.0) / 1e9
            scans[st_name] = {"GB/s": gbs, "frac_of_hbm": gbs / hbm, "algorithmic_bytes": per_rank}
    line = {
        "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong" if sp else "weak",
        "vs_baseline": None, "dtype": cfg["dtype"],
        "data": "synthetic (uniform q,k,v in [-1,1]" + (", gates in [0.9,1])" if cfg["gated"] else ", ungated)"),
        "config": {"workload": workload, **cfg,
                   "parallelism": (f"sequence chunk ranges over {world} rank(s), NCCL P2P carry chain" if sp
                                   else f"streams (b*h) per rank, {world} rank(s)"),
                   "l2": "inputs >= 512 MiB each >> 126 MB L2; no flush" if t * b * h * d >= 2 ** 28 else
                         "small config: inputs fit in L2 (no flush)"},
        "tflops_algorithmic": tflops, "frac_of_peak": tflops / peak, "frac_of_sustained_peak": tflops / peak_sus,
        "gpu_launches": launches, "stages_ms": stage_ms, "scans": scans, "clocks": ck, "e2e": e2e,
        "roofline": roof,
    }
    if world == 1 and not args.no_cpu:
        try:
            cores = os.cpu_count() or 1
            v, wall, desc = cpu_sample(cfg, cores)
            line["cpu_baseline"] = {"value": v, "unit": "tokens/s", "cores": cores, "kind": "port", "sample": desc,
                                    "sample_seconds": wall}
        except Exception as exc:  # the CPU leg must not sink the GPU number
            line["cpu_baseline"] = {"value": None, "error": repr(exc)}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


LM_WORKLOAD = ("configs[4]: 12-layer 124M power-attention LM (width 768, 12 heads d=64, MLP x4, tied 50257 "
               "embedding) fwd+bwd+AdamW, bf16 autocast, p=2 chunk=1024 gated, 32768-token sequence per GPU, "
               "data parallel (DDP bucketed NCCL all-reduce)")


def run_lm(args, world, rank, local):
    """configs[4]: one training step = forward + loss + backward (DDP all-reduce
    overlapped) + fused AdamW over one 32768-token sequence per GPU."""
    import torch
    import torch.distributed as dist

    from paper_2507_04239_b200 import _lib
    from paper_2507_04239_b200.lm import LMConfig, PowerLM, attention_flops, train_step, weight_flops

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    torch.manual_seed(0)
    cfg = LMConfig()
    t = 32768
    model = PowerLM(cfg).to(dev)
    net = model
    if world > 1:
        net = torch.nn.parallel.DistributedDataParallel(model, device_ids=[local], bucket_cap_mb=25,
                                                        gradient_as_bucket_view=True)
    opt = torch.optim.AdamW(model.parameters(), lr=3e-4, fused=True)
    g = torch.Generator(device=dev).manual_seed(100 + rank)
    tokens = torch.randint(0, cfg.vocab, (1, t + 1), device=dev, generator=g)
    x, y = tokens[:, :-1], tokens[:, 1:]

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    clocks = Clocks(local)
    clocks.start()
    for _ in range(args.warmup):
        train_step(net, opt, x, y)
    barrier()
    clocks.mark()
    _lib.profile_reset()
    _lib.profile_enable(True)
    n0 = _lib.launch_count()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        loss = train_step(net, opt, x, y)
    e1.record()
    barrier()
    launches = _lib.launch_count() - n0
    _lib.profile_enable(False)
    stages = _lib.profile_read()
    ck = clocks.stop()
    ms = e0.elapsed_time(e1) / args.steps
    if world > 1:
        tt = torch.tensor([ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    attn_ms = sum(v[0] for v in stages.values()) / args.steps

    # e2e: token ids from pinned host memory every step, the loss read back every step
    e2e = None
    if not args.no_e2e:
        host = tokens.cpu().pin_memory()
        dbuf = torch.empty_like(tokens)
        barrier()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record()
        ne = max(3, args.steps)
        for _ in range(ne):
            dbuf.copy_(host, non_blocking=True)
            lv = train_step(net, opt, dbuf[:, :-1], dbuf[:, 1:]).item()
        f1.record()
        barrier()
        ems = f0.elapsed_time(f1) / ne
        if world > 1:
            tt = torch.tensor([ems], device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ems = float(tt.item())
        e2e = {"value": world * t / (ems / 1000.0), "unit": "tokens/s",
               "h2d_bytes_per_step": host.numel() * host.element_size(), "d2h_bytes_per_step": 4,
               "ms_per_step": ems, "loss": lv}
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    peak, peak_sus, hbm, peak_kind = load_peaks()
    af = attention_flops(cfg, t)
    wf = weight_flops(cfg, t)
    tflops = world * (af + wf) / (ms / 1000.0) / 1e12
    attn_tflops = af / (attn_ms / 1000.0) / 1e12 if attn_ms > 0 else None
    line = {
        "metric": "LM training tokens/sec (configs[4]), whole job", "value": world * t / (ms / 1000.0),
        "unit": "tokens/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic uniform token ids, random-init weights",
        "config": {"workload": LM_WORKLOAD, "model": "power-attention GPT-2-small geometry", "global_batch": world,
                   "seq_len": t, "parallelism": f"dp{world}",
                   "params": sum(p.numel() for p in model.parameters())},
        "tflops_algorithmic": tflops, "frac_of_peak": tflops / peak,
        "attention": {"ms_per_step": attn_ms, "share_of_step": attn_ms / ms, "tflops_algorithmic": attn_tflops,
                      "frac_of_peak": attn_tflops / peak if attn_tflops else None,
                      "flops_share": af / (af + wf),
                      "stages_ms": {k: v[0] / args.steps for k, v in stages.items()}},
        "dense_layers": "torch nn.Linear / cuBLAS (outside the power-attention path)",
        "gpu_launches": launches, "clocks": ck, "e2e": e2e, "loss": float(loss),
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def stage_flops(stage: str, fl: dict):
    """Algorithmic FLOPs of one stage per step (the kernel's share of SURVEY 8d)."""
    return {
        "fwd_update_state": fl["update"],
        "fwd_attn_query": fl["intra"] + fl["query"],
        "bwd_attn_query": 2 * (fl["intra"] + fl["query"]),
        "bwd_update_state": 2 * fl["update"],
        "bwd_query_state": 2 * fl["query"],
        "bwd_intra": 2 * fl["intra"],
        "bwd_fp32": fl["bwd"],
    }.get(stage)


def traffic_for(stage: str):
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            return json.load(f).get(stage)
    except Exception:
        return None


def spawn_ranks(n: int) -> int:
    """`bench.py --gpus N` outside torchrun: re-launch under torch.distributed.run
    with one process per GPU (rendezvous on 127.0.0.1)."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--workload", default="auto", choices=["auto", *WORKLOADS, "lm124m"],
                    help="auto: cfg2 (BASELINE configs[1]) on one GPU, sp1m (configs[3], one 1M-token sequence "
                         "split over the ranks) on several; cfg1 / cfg3: configs[0] / configs[2]; lm124m: "
                         "configs[4], the 12-layer 124M power-attention LM, data parallel")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args.gpus))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
