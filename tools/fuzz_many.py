"""Wide one-off parity fuzz (robustness sweep beyond tests/test_fuzz_gpu.py): random fixed-length
and variable-length problems — MHA / GQA / MQA (including the grouped-query dK/dV split),
D 64 / 128, causal or not, [B,H,N,D] or [B,N,H,D] storage, random softmax_scale, uniform or
peaky inputs — forward O / L and backward dQ / dK / dV against the fp64 oracle.
Usage: python tools/fuzz_many.py [cases] [seed0]"""
import os
import random
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import oracle as orc  # noqa: E402
from paper_2410_20399_b200 import attention as A  # noqa: E402

MAX_ABS, REL_L2, L_ABS = 2e-2, 1e-2, 1e-3


def check(name, got, ref, tol=MAX_ABS):
    """The north-star bar (max-abs 2e-2, rel-L2 1e-2) is for O(1) outputs; peaky inputs, large
    scales and grouped-query sums make outputs of magnitude 4-10 whose bf16 rounding alone is
    0.015-0.03. So max-abs is held to max(2e-2, 2 bf16 ulps of the largest reference value),
    rel-L2 to 1e-2 unchanged; the plain north-star verdict is reported too."""
    got = np.asarray(got, dtype=np.float64)
    if not np.isfinite(got).all():
        return f"{name}: non-finite"
    ma, rl = orc.max_abs(got, ref), orc.rel_l2(got, ref)
    peak = float(np.abs(ref).max()) if np.size(ref) else 0.0
    ulps = ma / max(peak * 2.0 ** -8, 1e-30)
    if ma <= max(tol, 2.0 * 2.0 ** -8 * peak) and rl <= REL_L2:
        if ma > tol:
            NOTES.append(f"{name}: max-abs {ma:.3g} = {ulps:.2f} bf16 ulps of max |ref| {peak:.3g}")
        return None
    return f"{name}: max-abs {ma:.3g} ({ulps:.2f} ulps of max |ref| {peak:.3g}) rel-l2 {rl:.3g}"


NOTES = []


def run_case(seed):
    r = random.Random(seed)
    hkv = r.choice([1, 1, 2, 4])
    h = hkv * r.choice([1, 2, 4, 8])
    D = r.choice([64, 128])
    causal = r.random() < 0.5
    scale = r.choice([None, None, 0.05, 0.3])
    peaky = r.random() < 0.25
    varlen = r.random() < 0.3
    amp = 4.0 if peaky else 1.0
    if varlen:
        B = r.randint(1, 5)
        lens = [r.choice([0, 1, 37, 128, 129, 300, 640, 1000]) for _ in range(B)]
        if max(lens) == 0:
            lens[0] = 5
        T = sum(lens)
        q = orc.fill(seed, T * h * D).reshape(T, h, D) * amp
        k = orc.fill(seed + 1, T * hkv * D).reshape(T, hkv, D) * amp
        v = orc.fill(seed + 2, T * hkv * D).reshape(T, hkv, D)
        do = orc.fill(seed + 3, T * h * D).reshape(T, h, D)
        q, k = (np.asarray(x, dtype=np.float32).astype(np.float32) for x in (q, k))
        tq, tk, tv, tdo = (torch.from_numpy(np.ascontiguousarray(x)).to("cuda", torch.bfloat16) for x in (q, k, v, do))
        # the oracle sees the bf16-rounded values the GPU sees
        q, k, v, do = (t.float().cpu().numpy() for t in (tq, tk, tv, tdo))
        cu = torch.tensor(np.concatenate([[0], np.cumsum(lens)]), dtype=torch.int32, device="cuda")
        o, lse = A.attention_fwd_varlen(tq, tk, tv, cu, max(lens), causal=causal, softmax_scale=scale)
        dq, dk, dv = A.attention_bwd_varlen(tq, tk, tv, o, tdo, lse, cu, max(lens), causal=causal, softmax_scale=scale)
        torch.cuda.synchronize()
        o, dq, dk, dv = (t.float().cpu().numpy() for t in (o, dq, dk, dv))
        lse = lse.cpu().numpy()
        g = h // hkv
        s0 = 0
        for b, n in enumerate(lens):
            if n == 0:
                continue
            sl = slice(s0, s0 + n)
            s0 += n
            qh = np.transpose(q[sl], (1, 0, 2))
            kh = np.repeat(np.transpose(k[sl], (1, 0, 2)), g, axis=0)
            vh = np.repeat(np.transpose(v[sl], (1, 0, 2)), g, axis=0)
            doh = np.transpose(do[sl], (1, 0, 2))
            ro, rl = orc.attn_fwd(qh, kh, vh, causal=causal, scale=scale)
            rdq, rdk, rdv = orc.attn_bwd(qh, kh, vh, doh, causal=causal, scale=scale)
            rdk = rdk.reshape(hkv, g, n, D).sum(1)
            rdv = rdv.reshape(hkv, g, n, D).sum(1)
            for name, got, ref in (("o", np.transpose(o[sl], (1, 0, 2)), ro), ("dq", np.transpose(dq[sl], (1, 0, 2)), rdq),
                                   ("dk", np.transpose(dk[sl], (1, 0, 2)), rdk), ("dv", np.transpose(dv[sl], (1, 0, 2)), rdv)):
                err = check(name, got, ref)
                if err:
                    return f"varlen seq {b} n={n}: {err}"
            if orc.max_abs(lse[b, :, :n], rl) > L_ABS:
                return f"varlen seq {b}: lse"
        desc = f"varlen B{B} lens{lens}"
    else:
        B = r.randint(1, 3)
        N = r.choice([1, 17, 127, 128, 200, 384, 511, 1000, 1500])
        bnhd = r.random() < 0.3
        q = orc.fill(seed, B * h * N * D).reshape(B, h, N, D) * amp
        k = orc.fill(seed + 1, B * hkv * N * D).reshape(B, hkv, N, D) * amp
        v = orc.fill(seed + 2, B * hkv * N * D).reshape(B, hkv, N, D)
        do = orc.fill(seed + 3, B * h * N * D).reshape(B, h, N, D)

        def dev(x):
            t = torch.from_numpy(np.ascontiguousarray(x)).to("cuda", torch.bfloat16)
            return t.transpose(1, 2).contiguous().transpose(1, 2) if bnhd else t

        tq, tk, tv, tdo = (dev(x) for x in (q, k, v, do))
        q, k, v, do = (t.float().cpu().numpy() for t in (tq, tk, tv, tdo))
        o, lse = A.attention_fwd(tq, tk, tv, causal=causal, softmax_scale=scale)
        dq, dk, dv = A.attention_bwd(tq, tk, tv, o, tdo, lse, causal=causal, softmax_scale=scale)
        torch.cuda.synchronize()
        g = h // hkv
        ke = np.repeat(k, g, axis=1).reshape(-1, N, D)
        ve = np.repeat(v, g, axis=1).reshape(-1, N, D)
        ro, rl = orc.attn_fwd(q.reshape(-1, N, D), ke, ve, causal=causal, scale=scale)
        rdq, rdk, rdv = orc.attn_bwd(q.reshape(-1, N, D), ke, ve, do.reshape(-1, N, D), causal=causal, scale=scale)
        rdk = rdk.reshape(B, hkv, g, N, D).sum(2).reshape(-1, N, D)
        rdv = rdv.reshape(B, hkv, g, N, D).sum(2).reshape(-1, N, D)
        for name, got, ref in (("o", o, ro), ("dq", dq, rdq), ("dk", dk, rdk), ("dv", dv, rdv)):
            err = check(name, got.float().cpu().numpy().reshape(-1, N, D), ref)
            if err:
                return err
        if orc.max_abs(lse.cpu().numpy().reshape(-1, N), rl) > L_ABS:
            return "lse"
        desc = f"B{B} N{N}{' bnhd' if bnhd else ''}"
    return f"ok {desc} H{h} Hkv{hkv} D{D} c{int(causal)} scale={scale} peaky={peaky}"


if __name__ == "__main__":
    cases = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    seed0 = int(sys.argv[2]) if len(sys.argv) > 2 else 50000
    bad = 0
    for i in range(cases):
        res = run_case(seed0 + i)
        if not res.startswith("ok"):
            bad += 1
            print(f"case {seed0 + i}: FAIL {res}", flush=True)
    print(f"fuzz_many: {cases} cases, {bad} failures; {len(NOTES)} checks above the fixed 2e-2 bar but within "
          f"2 bf16 ulps of the output's magnitude:", flush=True)
    for nt in NOTES:
        print("   ", nt)
