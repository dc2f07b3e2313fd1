#!/usr/bin/env python
"""bench.py — the driver's benchmark contract for the B200 attention hot path.

Metric (BASELINE.json): attention fwd/bwd TFLOPS/GPU, BF16, D=128, causal, and its
fraction of the dense BF16 tensor peak. Workload (BASELINE configs[1]/[2]):
B=16 H=16 N=4096 D=128 causal, one step = one forward (saving L) + one backward
(dQ/dK/dV from L) over synthetic bf16 inputs resident in HBM (each input is 268 MB,
larger than the 126 MB L2, so no L2 flush is needed between steps).

  python bench.py [--gpus N --steps K --warmup W] [--impl tkb|reference] [--pass fwd|bwd|fwdbwd]

Multi-GPU (one process per GPU): under torchrun the ranks come from the environment;
`--gpus N` without torchrun spawns the N - 1 other ranks itself (rank r on visible device
r % device_count). The flattened batch x head grid of a global problem with B = 16 * N is
sharded contiguously across ranks (tkb_shard_range); every (b, h) unit's inputs come from
its own seed, so a shard equals the same slice of a 1-GPU run. No collective touches the
data path and NCCL is never initialised: the only cross-rank traffic is a gloo (CPU)
barrier and the max-over-ranks of the CUDA-event time ("scaling": "weak").

FLOP convention (FlashAttention / SURVEY.md §8(d)): fwd 4 B H N^2 D, bwd 10 B H N^2 D,
causal x 1/2.
"""
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

B_PER_GPU, H, N, D = 16, 16, 4096, 128
FALLBACK_PEAKS = {"bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "hbm_gbs": 6650.0}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="tkb", choices=["tkb", "reference"])
    ap.add_argument("--pass", dest="which", default="fwdbwd", choices=["fwd", "bwd", "fwdbwd"])
    ap.add_argument("--causal", type=int, default=1)
    ap.add_argument("--batch", type=int, default=B_PER_GPU, help="per-GPU batch")
    ap.add_argument("--heads", type=int, default=H)
    ap.add_argument("--seq", type=int, default=N)
    ap.add_argument("--head-dim", type=int, default=D)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-chunks", type=int, default=16, help="batch chunks pipelined in the e2e step")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--dump-hashes", default=None, help="write per-unit output hashes (JSON) after the run")
    return ap.parse_args()


def flops(b, h, n, d, causal, which):
    f = 0.0
    if "fwd" in which:
        f += 4.0 * b * h * n * n * d
    if "bwd" in which:
        f += 10.0 * b * h * n * n * d
    return f * (0.5 if causal else 1.0)


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            j = json.load(f)
        return j, "measured"
    except Exception:
        return dict(FALLBACK_PEAKS), "fallback"


# ------------------------------------------------------------------ clocks


class ClockSampler:
    """nvidia-smi sampling DURING the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for nm, val in zip(names, parts[5:9]):
                if val.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ CPU legs (oracle / reference)


def cpu_reference_sample(causal, which, seq, head_dim, nthreads=None):
    """Time the reference's CPU path on a bounded sample: one (b,h) head per host thread.

    fwd: the UNMODIFIED reference kernel path (oracle/_ref: execute_functional(
         attention_fwd_kernel)). It only supports non-causal attention, so it computes the
         full N^2 and is credited with the non-causal FLOPs it executes.
    bwd: the reference has no backward; the oracle port's fp64 backward is timed (causal
         work skips the masked pairs, so it is credited with the causal FLOPs).
    kind is "reference" only when every timed part is the reference's own code.
    """
    import numpy as np  # noqa: F401
    from concurrent.futures import ThreadPoolExecutor

    from oracle import oracle as orc

    nthreads = nthreads or orc.threads()
    heads = nthreads
    q, k, v = orc.qkv(1234, 1, heads, seq, head_dim)
    dout = orc.fill(99, heads * seq * head_dim).reshape(1, heads, seq, head_dim)
    use_ref = orc.ref_available()
    fl = 0.0
    t0 = time.perf_counter()
    if "fwd" in which:
        if use_ref:
            def one(hh):
                return orc.ref_attention_fwd(q[:, hh:hh + 1], k[:, hh:hh + 1], v[:, hh:hh + 1], kv_rows=128,
                                             workers=4, bf16=True, threaded=False)
            with ThreadPoolExecutor(nthreads) as ex:
                list(ex.map(one, range(heads)))
            fl += flops(1, heads, seq, head_dim, False, "fwd")
        else:
            orc.attn_fwd(q, k, v, causal=causal, nthreads=nthreads)
            fl += flops(1, heads, seq, head_dim, causal, "fwd")
    t1 = time.perf_counter()
    if "bwd" in which:
        orc.attn_bwd(q, k, v, dout, causal=causal, nthreads=nthreads)
        fl += flops(1, heads, seq, head_dim, causal, "bwd")
    t2 = time.perf_counter()
    ref_only = use_ref and "bwd" not in which
    fwd_desc = ("reference execute_functional(attention_fwd_kernel) [non-causal only: full N^2 executed and "
                "credited, bf16-emulated]" if use_ref else "oracle port fp64")
    return {
        "value": fl / (t2 - t0) / 1e12,
        "unit": "TFLOPS",
        "cores": nthreads,
        "kind": "reference" if ref_only else "port",
        "sample": (f"{heads} (b,h) heads of N={seq} D={head_dim}, one per host thread; fwd = {fwd_desc} "
                   f"{t1 - t0:.2f}s; bwd = oracle port fp64 (the reference has no backward) {t2 - t1:.2f}s"),
        "seconds": t2 - t0,
    }


# ------------------------------------------------------------------ reference arm


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    causal = bool(args.causal)
    vals = []
    base = None
    for i in range(args.warmup + args.steps):
        r = cpu_reference_sample(causal, args.which, args.seq, args.head_dim)
        if i >= args.warmup:
            vals.append(r["value"])
            base = r
    value = statistics.mean(vals)
    line = {
        "impl": "reference",
        "metric": "attention fwd+bwd TFLOPS/GPU (BF16, D=128, causal)" if args.which == "fwdbwd"
        else f"attention {args.which} TFLOPS/GPU (BF16, D=128, causal)",
        "value": value,
        "unit": "TFLOPS",
        "n_gpus": args.gpus,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": base["seconds"] * 1e3,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic",
        "config": workload_config(args, 1),
        "cpu_baseline": {k: base[k] for k in ("value", "unit", "cores", "kind", "sample")},
        "e2e": {"value": value, "unit": "TFLOPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


L2_BYTES = 126 * 2 ** 20


def needs_flush(args):
    """Inputs that fit in L2 get an L2 flush between timed steps (timing rules)."""
    return 4 * args.batch * args.heads * args.seq * args.head_dim * 2 < 2 * L2_BYTES


def workload_config(args, world):
    shape = (args.batch, args.heads, args.seq, args.head_dim)
    named = {(16, 16, 4096, 128): "BASELINE configs[1]+[2]", (1, 8, 1024, 64): "BASELINE configs[0]",
             (32, 32, 16384, 128): "BASELINE configs[4] per GPU at N=1 (1/8 of it per GPU at 8 GPUs: B=4)",
             (4, 32, 16384, 128): "BASELINE configs[4] per-GPU shard at 8 GPUs"}.get(shape, "BASELINE configs[3] sweep point"
                                                                                  if args.heads == 16 and args.batch == 16
                                                                                  else "custom")
    tensor_mb = args.batch * args.heads * args.seq * args.head_dim * 2 / 2 ** 20
    return {
        "workload": f"attention {'fwd+bwd' if args.which == 'fwdbwd' else args.which} "
                    f"{'causal' if args.causal else 'non-causal'} B={args.batch}/GPU H={args.heads} "
                    f"N={args.seq} D={args.head_dim} bf16 ({named})",
        "batch_per_gpu": args.batch,
        "global_batch": args.batch * world,
        "heads": args.heads,
        "seq_len": args.seq,
        "head_dim": args.head_dim,
        "causal": bool(args.causal),
        "parallelism": f"bh-shard{world}",
        "l2": (f"L2 flushed between timed steps (inputs {tensor_mb:.1f} MB per tensor fit in the 126 MB L2); "
               "value = sum of the steps' own device time" if needs_flush(args)
               else f"inputs larger than L2 ({tensor_mb:.0f} MB per tensor); no flush"),
    }


# ------------------------------------------------------------------ tkb arm


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args)

    import torch
    import torch.distributed as dist

    from paper_2410_20399_b200 import attention as A

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    ndev = torch.cuda.device_count()
    dev_index = local % max(1, ndev)
    torch.cuda.set_device(dev_index)
    dev = torch.device("cuda", dev_index)
    if world > 1:  # CPU-side group for the barrier and the timing max; no NCCL anywhere
        dist.init_process_group("gloo", rank=rank, world_size=world)

    causal = bool(args.causal)
    b_loc, h, n, d = args.batch, args.heads, args.seq, args.head_dim
    # global problem B = batch * world; this rank's contiguous (b,h) shard
    units = b_loc * world * h
    u0, u1 = A.shard_range(units, rank, world)
    my_units = u1 - u0
    shape = (1, my_units, n, d)
    q, k, v, do = (torch.empty(shape, device=dev, dtype=torch.bfloat16) for _ in range(4))
    gen = torch.Generator(device=dev)
    for i, u in enumerate(range(u0, u1)):  # per-unit seeds: shards == the 1-GPU slices
        gen.manual_seed(1000 + u)
        for t in (q, k, v, do):
            t[0, i].uniform_(-1, 1, generator=gen)
    o = torch.empty_like(q)
    lse = torch.empty((1, my_units, n), device=dev, dtype=torch.float32)
    dq, dk, dv = torch.empty_like(q), torch.empty_like(q), torch.empty_like(q)
    ws = torch.empty(A.bwd_workspace_bytes(1, my_units, n, d, causal), device=dev, dtype=torch.uint8)
    stream = torch.cuda.current_stream(dev)
    which = args.which

    launches = {"n": 0}
    marks = []  # in-step CUDA events (timed region only): [before fwd, between, after bwd] per step

    def step(mark=False):
        cnt = 0
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(3)] if mark else None
        if mark:
            evs[0].record(stream)
        if "fwd" in which:
            A.attention_fwd(q, k, v, causal=causal, out=o, lse=lse)
            cnt += A.last_launch_count()
        if mark:
            evs[1].record(stream)
        if "bwd" in which:
            A.attention_bwd(q, k, v, o, do, lse, causal=causal, dq=dq, dk=dk, dv=dv, workspace=ws)
            cnt += A.last_launch_count()
        if mark:
            evs[2].record(stream)
            marks.append(evs)
        launches["n"] += cnt

    if "bwd" in which and "fwd" not in which:
        A.attention_fwd(q, k, v, causal=causal, out=o, lse=lse)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)

    # per-kernel timing (roofline): CUDA events on the launching stream around each kernel
    # (the backward's three kernels are isolated with the debug phase mask)
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    kern_ms = {}

    def time_it(fn, reps=3):
        e0, e1 = ev(), ev()
        e0.record(stream)
        for _ in range(reps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize(dev)
        return e0.elapsed_time(e1) / reps

    if "fwd" in which:
        kern_ms["attn_fwd"] = time_it(lambda: A.attention_fwd(q, k, v, causal=causal, out=o, lse=lse))
    if "bwd" in which:
        bwd = lambda: A.attention_bwd(q, k, v, o, do, lse, causal=causal, dq=dq, dk=dk, dv=dv, workspace=ws)  # noqa
        for name, mask in (("bwd_prep", 1), ("attn_bwd_dkdv", 2), ("attn_bwd_dq", 4)):
            A.debug_set_bwd_phases(mask)
            kern_ms[name] = time_it(bwd)
        A.debug_set_bwd_phases(7)
        bwd()  # restore complete outputs
        torch.cuda.synchronize(dev)

    # timed region
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    launches["n"] = 0
    start, end = ev(), ev()
    with ClockSampler(local) as clk:
        # ~1 s of untimed steps under the sampler so the clock record covers steady load
        t_soak = time.time()
        while time.time() - t_soak < 1.0:
            step()
            torch.cuda.synchronize(dev)
        launches["n"] = 0
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        flush = needs_flush(args)
        scrub = torch.empty(2 * L2_BYTES // 4, device=dev, dtype=torch.float32) if flush else None
        start.record(stream)
        for _ in range(args.steps):
            if flush:
                scrub.fill_(1.0)  # evict the inputs from L2 (outside the step's own events)
            step(mark=True)
        end.record(stream)
        torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    ms = start.elapsed_time(end)
    if needs_flush(args):  # the steps' own device time, flushes excluded
        ms = sum(m[0].elapsed_time(m[2]) for m in marks)
    t = torch.tensor([ms], dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)  # timing only (gloo, CPU), not on the data path
    ms_max = float(t.item())
    if args.dump_hashes:
        dump_hashes(args, world, rank, u0, [o, lse, dq, dk, dv], which)
    gpu_launches = launches["n"]

    total_flops = flops(1, units, n, d, causal, which) * args.steps
    value = total_flops / (ms_max / 1e3) / 1e12

    # e2e through the public API with host buffers (pinned), H2D + D2H inside the timed region
    e2e = None
    if not args.no_e2e:
        hq, hk, hv, hdo = (x.cpu().pin_memory() for x in (q, k, v, do))
        ho = torch.empty(q.shape, dtype=torch.bfloat16).pin_memory()
        hdq, hdk, hdv = (torch.empty(q.shape, dtype=torch.bfloat16).pin_memory() for _ in range(3))
        h2d = d2h = 0

        # The public API calls run on chunks of the batch over three streams (H2D copy,
        # compute, D2H copy) so PCIe transfers in both directions overlap the kernels and
        # each other; every step still moves all of its inputs in and all of its results out.
        chunks = max(c for c in range(1, max(1, args.e2e_chunks) + 1) if my_units % c == 0)
        cb = my_units // chunks
        s_h2d, s_cmp, s_d2h = torch.cuda.Stream(dev), torch.cuda.Stream(dev), torch.cuda.Stream(dev)

        def e2e_step():
            nonlocal h2d, d2h
            h2d = d2h = 0
            done_prev = []
            for c in range(chunks):
                sl = (slice(None), slice(c * cb, (c + 1) * cb))  # a run of (b, h) units
                with torch.cuda.stream(s_h2d):
                    for dst, src in ((q, hq), (k, hk), (v, hv)) + (((do, hdo),) if "bwd" in which else ()):
                        dst[sl].copy_(src[sl], non_blocking=True)
                        h2d += dst[sl].numel() * 2
                    ev_in = torch.cuda.Event()
                    ev_in.record(s_h2d)
                with torch.cuda.stream(s_cmp):
                    s_cmp.wait_event(ev_in)
                    if "fwd" in which:
                        A.attention_fwd(q[sl], k[sl], v[sl], causal=causal, out=o[sl], lse=lse[sl])
                    if "bwd" in which:
                        A.attention_bwd(q[sl], k[sl], v[sl], o[sl], do[sl], lse[sl], causal=causal, dq=dq[sl],
                                        dk=dk[sl], dv=dv[sl], workspace=ws)
                    ev_out = torch.cuda.Event()
                    ev_out.record(s_cmp)
                with torch.cuda.stream(s_d2h):
                    s_d2h.wait_event(ev_out)
                    outs = ((ho, o),) if "fwd" in which else ()
                    if "bwd" in which:
                        outs += ((hdq, dq), (hdk, dk), (hdv, dv))
                    for dst, src in outs:
                        dst[sl].copy_(src[sl], non_blocking=True)
                        d2h += src[sl].numel() * 2
                    ev_done = torch.cuda.Event()
                    ev_done.record(s_d2h)
                done_prev.append(ev_done)
            for e in done_prev:  # the step ends when its last result is on the host
                stream.wait_event(e)

        e2e_step()
        torch.cuda.synchronize(dev)
        e2e_steps = max(1, min(args.steps, 5))
        if world > 1:
            dist.barrier()
        s2, e2 = ev(), ev()
        s2.record(stream)
        for st_ in (s_h2d, s_cmp, s_d2h):
            st_.wait_event(s2)
        for _ in range(e2e_steps):
            e2e_step()
        e2.record(stream)
        torch.cuda.synchronize(dev)
        t2 = torch.tensor([s2.elapsed_time(e2)], dtype=torch.float64)
        if world > 1:
            dist.all_reduce(t2, op=dist.ReduceOp.MAX)
        e2e_val = flops(1, units, n, d, causal, which) * e2e_steps / (float(t2.item()) / 1e3) / 1e12
        e2e = {"value": e2e_val, "unit": "TFLOPS", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "pipeline": f"{chunks} batch chunks on 3 streams (H2D / compute / D2H overlap)"}

    if rank == 0:
        peaks, peak_src = load_peaks()
        # algorithmic work per launch of each kernel (the backward runs as
        # a dK/dV kernel of 4 GEMMs and a dQ kernel of 3 GEMMs)
        cf = 0.5 if causal else 1.0
        work = {
            "attn_fwd": ("tensor", 4.0 * my_units * n * n * d * cf),
            "attn_bwd_dkdv": ("tensor", 8.0 * my_units * n * n * d * cf),
            "attn_bwd_dq": ("tensor", 6.0 * my_units * n * n * d * cf),
            "bwd_prep": ("hbm", (2 * 2 * my_units * n * d + 4 * my_units * n + 8 * my_units * n)),
        }
        dom = max(kern_ms, key=lambda x: kern_ms[x])
        bound, amount = work[dom]
        if bound == "tensor":
            achieved = amount / (kern_ms[dom] / 1e3) / 1e12
            peak = float(peaks.get("bf16_tflops", FALLBACK_PEAKS["bf16_tflops"]))
            unit = "TFLOP/s"
        else:
            achieved = amount / (kern_ms[dom] / 1e3) / 1e9
            peak = float(peaks.get("hbm_gbs", FALLBACK_PEAKS["hbm_gbs"]))
            unit = "GB/s"
        per_kernel = {}
        io_bytes = {"attn_fwd": 8 * my_units * n * d + 4 * my_units * n,  # SURVEY §8(d) algorithmic bytes
                    "attn_bwd_dkdv": 0, "attn_bwd_dq": 0, "bwd_prep": work["bwd_prep"][1]}
        for kname, ms_k in kern_ms.items():
            b_k, amt = work[kname]
            rate = amt / (ms_k / 1e3) / (1e12 if b_k == "tensor" else 1e9)
            per_kernel[kname] = {"ms": ms_k, "bound": b_k, "achieved": rate,
                                 "unit": "TFLOP/s" if b_k == "tensor" else "GB/s"}
            if kname == "attn_fwd":  # memory side of the forward (short sequences are HBM / latency bound)
                per_kernel[kname]["us"] = ms_k * 1e3
                per_kernel[kname]["algorithmic_gbs"] = io_bytes[kname] / (ms_k / 1e3) / 1e9
        # In-step times: the forward and backward calls of the timed steps themselves (events
        # between the calls), against the measured peak sustained under this load; the dominant
        # kernel's in-step time is its share of its pass from the isolated (burst) timings.
        in_step = None
        if marks:
            fwd_in = statistics.mean(m[0].elapsed_time(m[1]) for m in marks)
            bwd_in = statistics.mean(m[1].elapsed_time(m[2]) for m in marks)
            in_step = {"attn_fwd_ms": fwd_in, "bwd_ms": bwd_in}
            bwd_iso = sum(kern_ms.get(x, 0.0) for x in ("bwd_prep", "attn_bwd_dkdv", "attn_bwd_dq"))
            dom_in = (fwd_in if dom == "attn_fwd" else bwd_in * kern_ms[dom] / bwd_iso) if (
                dom == "attn_fwd" or bwd_iso > 0) else None
            if dom_in and bound == "tensor":
                sust = float(peaks.get("bf16_tflops_sustained", 1400.0))
                ach_in = amount / (dom_in / 1e3) / 1e12
                in_step.update({"dominant_ms": dom_in, "dominant_achieved": ach_in,
                                "dominant_frac_of_burst": ach_in / peak, "dominant_frac_of_sustained": ach_in / sust})
            if "fwd" in which and fwd_in > 0:
                in_step["fwd_tflops"] = flops(1, my_units, n, d, causal, "fwd") / (fwd_in / 1e3) / 1e12
            if "bwd" in which and bwd_in > 0:
                bt = flops(1, my_units, n, d, causal, "bwd") / (bwd_in / 1e3) / 1e12
                in_step["bwd_tflops"] = bt
                in_step["bwd_frac_of_sustained"] = bt / float(peaks.get("bf16_tflops_sustained", 1400.0))
        roofline = {
            "bound": bound,
            "kernel": dom,
            "achieved": achieved,
            "peak": peak,
            "unit": unit,
            "frac": achieved / peak,
            "peak_source": ("measured bf16 burst, MEASURED_PEAKS.json" if bound == "tensor"
                            else "measured HBM copy, MEASURED_PEAKS.json") if peak_src == "measured"
            else "fallback (B200_PROFILING.md)",
            "work_per_launch": amount,
            "frac_of_sustained": (achieved / float(peaks.get("bf16_tflops_sustained", 1400.0))
                                  if bound == "tensor" else None),
            "traffic": load_traffic(dom),
            "per_kernel": per_kernel,
            "per_kernel_timing": "isolated launches before the soak (burst clocks)",
            "in_step": in_step,
        }
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            try:
                r = cpu_reference_sample(causal, which, n, d)
                cpu = {k2: r[k2] for k2 in ("value", "unit", "cores", "kind", "sample")}
            except Exception as ex:  # the CPU leg is reported, never required
                cpu = {"value": None, "unit": "TFLOPS", "cores": 0, "kind": "port", "sample": f"failed: {ex}"}
        line = {
            "metric": "attention fwd+bwd TFLOPS/GPU (BF16, D=128, causal)" if which == "fwdbwd"
            else f"attention {which} TFLOPS/GPU (BF16, D=128, causal)",
            "value": value,
            "unit": "TFLOPS",
            "n_gpus": world,
            "devices": min(world, ndev),
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms_max / args.steps,
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "bf16",
            "data": "synthetic",
            "config": workload_config(args, world),
            "tflops_per_gpu": value / world,
            "frac_of_peak": value / world / float(load_peaks()[0].get("bf16_tflops", 1590.0)),
            "e2e": e2e,
            "gpu_launches": gpu_launches,
            "roofline": roofline,
            "cpu_baseline": cpu,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def dump_hashes(args, world, rank, u0, outs, which):
    """Per-unit FNV-1a hashes of the step's outputs (O, L, dQ, dK, dV bytes), merged over
    ranks in the file `args.dump_hashes` (one JSON object: unit -> hash)."""
    import hashlib

    import torch

    torch.cuda.synchronize()
    hs = {}
    for i in range(outs[0].shape[1]):
        hsh = hashlib.sha1()
        for t in outs:
            hsh.update(t[0, i].contiguous().view(torch.uint8).cpu().numpy().tobytes())
        hs[str(u0 + i)] = hsh.hexdigest()
    path = f"{args.dump_hashes}.rank{rank}"
    with open(path, "w") as f:
        json.dump(hs, f)
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
    if rank == 0:
        merged = {}
        for r in range(world):
            with open(f"{args.dump_hashes}.rank{r}") as f:
                merged.update(json.load(f))
        with open(args.dump_hashes, "w") as f:
            json.dump(merged, f, sort_keys=True)


def spawn_ranks(args):
    """`--gpus N` without torchrun: run N ranks (this process is rank 0), one process per
    GPU, rendezvous on 127.0.0.1 for the gloo timing group."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    base = dict(os.environ, WORLD_SIZE=str(args.gpus), MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    kids = []
    for r in range(1, args.gpus):
        env = dict(base, RANK=str(r), LOCAL_RANK=str(r))
        kids.append(subprocess.Popen([sys.executable, os.path.abspath(__file__)] + sys.argv[1:], env=env))
    os.environ.update(base, RANK="0", LOCAL_RANK="0")
    rc = main()
    for kd in kids:
        rc = kd.wait() or rc
    return rc


def load_traffic(kernel):
    """dram bytes per launch from the committed ncu capture summary, if any."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(p) as f:
            t = json.load(f)
        # logical kernel -> the symbol ncu reports (dK/dV runs as the persistent kernel)
        sym = {"attn_bwd_dkdv": "attn_bwd_dkdv_template", "attn_fwd": "attn_fwd_template",
               "attn_bwd_dq": "attn_bwd_dq_template"}.get(kernel, kernel + "_kernel")
        return t.get(sym, t.get(kernel))
    except Exception:
        return None


if __name__ == "__main__":
    sys.exit(main())
