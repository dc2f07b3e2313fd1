import sys, os, time, subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if len(sys.argv) > 1 and sys.argv[1] == "one":
    import torch
    from paper_2410_20399_b200 import attention as A
    B, H, N, D, causal = map(int, sys.argv[2:7])
    q, k, v, do = (torch.randn(B, H, N, D, device="cuda", dtype=torch.bfloat16) for _ in range(4))
    o, lse = A.attention_fwd(q, k, v, causal=bool(causal))
    torch.cuda.synchronize()
    t0 = time.time()
    A.attention_bwd(q, k, v, o, do, lse, causal=bool(causal))
    torch.cuda.synchronize()
    t1 = time.time()
    A.attention_bwd(q, k, v, o, do, lse, causal=bool(causal))
    torch.cuda.synchronize()
    print(f"B{B} H{H} N{N} D{D} c{causal}: first {1e3*(t1-t0):.2f} ms, second {1e3*(time.time()-t1):.2f} ms", flush=True)
    sys.exit(0)
for shape in sys.argv[1].split(";"):
    try:
        r = subprocess.run([sys.executable, __file__, "one"] + shape.split(","), timeout=40, capture_output=True, text=True)
        print(r.stdout.strip() or r.stderr.strip()[-300:], flush=True)
    except subprocess.TimeoutExpired:
        print(shape, "TIMEOUT", flush=True)
