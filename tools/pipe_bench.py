"""Per-SM throughput of the softmax building blocks (MUFU ex2, bf16 pack, FFMA, f32x2, poly exp2)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2410_20399_b200 import _lib
L = _lib.load_selftest()
f = L.tkb_selftest_pipe_bench
f.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
out = torch.zeros(256, device="cuda")
cyc = torch.zeros(1, dtype=torch.int64, device="cuda")
names = ["ex2.approx", "cvt bf16x2", "ex2+cvt", "ffma", "fma.f32x2", "poly3 exp2 (f32x2)"]
per_iter = [16, 8, 16, 16, 16, 16]   # elements (or pairs for cvt) per thread per iteration
for mode, nm in enumerate(names):
    iters = 2000
    f(out.data_ptr(), mode, iters, cyc.data_ptr(), None)
    torch.cuda.synchronize()
    f(out.data_ptr(), mode, iters, cyc.data_ptr(), None)
    torch.cuda.synchronize()
    ops = 256 * iters * per_iter[mode]
    print(f"{nm:20s}: {ops / cyc.item():6.1f} elements/clk per SM (256 threads)")
