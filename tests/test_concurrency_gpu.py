"""The ABI's concurrency contract (include/tkb_attn.h): calls are asynchronous on the caller's
stream and safe from several host threads on any mix of streams. The persistent kernels claim
tasks from a per-(device, stream) counter slot, so kernels running at the same time on
different streams must not share a queue; and a call after tkb_device_init() is capturable in
a CUDA graph. Every concurrent / captured result must equal the plain sequential one bit for bit
(the kernels are deterministic)."""
import threading

import pytest
import torch

from paper_2410_20399_b200 import attention as A

pytestmark = pytest.mark.gpu

B, H, N, D = 2, 4, 1024, 128


def _inputs(seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return [torch.empty((B, H, N, D), device="cuda", dtype=torch.bfloat16).uniform_(-1, 1, generator=g)
            for _ in range(4)]


def _step(q, k, v, do, causal=True):
    o, lse = A.attention_fwd(q, k, v, causal=causal)
    dq, dk, dv = A.attention_bwd(q, k, v, o, do, lse, causal=causal)
    return o, lse, dq, dk, dv


def _assert_equal(a, b):
    for x, y in zip(a, b):
        assert torch.equal(x, y)


def test_concurrent_streams(cuda_dev):
    inputs = [_inputs(100 + i) for i in range(4)]
    ref = [_step(*x) for x in inputs]
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream() for _ in inputs]
    for _ in range(3):  # the four steps overlap on the GPU (each kernel is one CTA per SM)
        out = []
        for s, x in zip(streams, inputs):
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                out.append(_step(*x))
        torch.cuda.synchronize()
        for r, o in zip(ref, out):
            _assert_equal(r, o)


def test_concurrent_host_threads(cuda_dev):
    inputs = [_inputs(200 + i) for i in range(3)]
    ref = [_step(*x) for x in inputs]
    torch.cuda.synchronize()
    results, errors = [None] * len(inputs), []

    def run(i):
        try:
            torch.cuda.set_device(0)
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                outs = [_step(*inputs[i]) for _ in range(3)]
            s.synchronize()
            results[i] = outs
        except Exception as e:  # noqa: BLE001 - reported below
            errors.append(e)

    threads = [threading.Thread(target=run, args=(i,)) for i in range(len(inputs))]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    for r, outs in zip(ref, results):
        for o in outs:
            _assert_equal(r, o)


def test_cuda_graph_capture(cuda_dev):
    A.device_init(0)  # the counter pool exists before capture: the captured calls allocate nothing
    q, k, v, do = _inputs(300)
    ws = torch.empty(A.bwd_workspace_bytes(B, H, N, D), dtype=torch.uint8, device="cuda")
    o, lse = torch.empty_like(q), torch.empty((B, H, N), dtype=torch.float32, device="cuda")
    dq, dk, dv = (torch.empty_like(q) for _ in range(3))

    def step():
        A.attention_fwd(q, k, v, causal=True, out=o, lse=lse)
        A.attention_bwd(q, k, v, o, do, lse, causal=True, dq=dq, dk=dk, dv=dv, workspace=ws)

    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        step()  # warm-up on the capture stream (TMA descriptor cache, smem opt-in)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        step()
    for seed in (301, 302, 303):
        for dst, src in zip((q, k, v, do), _inputs(seed)):
            dst.copy_(src)
        graph.replay()
        torch.cuda.synchronize()
        ref = _step(q, k, v, do)
        torch.cuda.synchronize()
        _assert_equal(ref, (o, lse, dq, dk, dv))


def test_cuda_graph_capture_rotary_forward(cuda_dev):
    """The fused rotary forward publishes per-block flags that its load warp waits on; they are
    cleared on the stream before each launch (a memset node in the graph), so every replay on
    new inputs waits for its own rotated blocks. A per-call epoch frozen into the graph would
    let replays 2+ read the previous replay's rotated Q / K."""
    A.device_init(0)
    q, k, v, _ = _inputs(400)
    pos = torch.arange(N, device="cuda", dtype=torch.float64)[:, None]
    freq = 10000.0 ** (-torch.arange(D // 2, device="cuda", dtype=torch.float64) / (D // 2))
    sin, cos = (f(pos * freq[None, :]).float().contiguous() for f in (torch.sin, torch.cos))
    o, lse = torch.empty_like(q), torch.empty((B, H, N), dtype=torch.float32, device="cuda")

    def step():
        return A.attention_fwd(q, k, v, causal=True, out=o, lse=lse, rotary_tables=(sin, cos), return_rotated=True)

    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        step()
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        _, _, q_rot, k_rot = step()
    for seed in (401, 402, 403):
        for dst, src in zip((q, k, v), _inputs(seed)):
            dst.copy_(src)
        graph.replay()
        torch.cuda.synchronize()
        qr, kr = A.rotary_qk(q, k, sin, cos)
        o_ref, l_ref = A.attention_fwd(qr, kr, v, causal=True)
        torch.cuda.synchronize()
        _assert_equal((qr, kr, o_ref, l_ref), (q_rot, k_rot, o, lse))
