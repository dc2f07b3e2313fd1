"""Chip-wide fp32 reduce-add throughput into L2 (the bwd dQ accumulation path)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2410_20399_b200 import _lib
L = _lib.load_selftest()
f = L.tkb_selftest_reduce_bench
f.argtypes = [ctypes.c_void_p] + [ctypes.c_int] * 5 + [ctypes.c_void_p]
region_chunks = 64 * 64  # 64 MB
g = torch.zeros(region_chunks * 4096, device="cuda")
for mode, name in ((0, "tma-tensor"), (1, "bulk-1d"), (2, "red.v4")):
    for inflight in ((1, 2, 4) if mode < 2 else (1,)):
        for ctas in (148, 296):
            iters = 200
            st = torch.cuda.current_stream().cuda_stream
            f(g.data_ptr(), mode, ctas, 20, inflight, region_chunks, st)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); f(g.data_ptr(), mode, ctas, iters, inflight, region_chunks, st); e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            gbs = ctas * iters * 16384 / ms / 1e6
            print(f"{name:11s} inflight={inflight} ctas={ctas}: {gbs:8.1f} GB/s  ({gbs/ctas:.1f} GB/s per CTA)", flush=True)
