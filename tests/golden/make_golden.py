"""Generate the golden fixtures that pin the CPU oracle to the reference.

Runs the UNMODIFIED reference attention path (kittensim, compiled from
/root/reference/proj/include into oracle/_ref/ by oracle/Makefile) on the reference's
own test cases and stores its outputs:

  attention_fwd_kernel + execute_functional     kernels.hpp:250-355, lcsf.hpp:779-819
  oracle_attention (fp64)                       oracles.hpp:34-64
  fill_uniform (std::mt19937 + U(-1,1))         report.hpp:57-61

Cases (reference test -> fixture key):
  test_kernels.cpp:110-126  constant V columns          const_v
  test_kernels.cpp:128-146  dense oracle, d=64 / 128     dense_d64, dense_d128
  test_kernels.cpp:148-170  KV-chunk invariance         chunk_kv384 / 192 / 128
  test_kernels.cpp:183-213  B=H=2 multi-head            bh2
  BASELINE configs[0]       B1 H8 N1024 D64 bf16 inputs  c1 (heads 0 and 7 stored)

Run here (needs /root/reference): python tests/golden/make_golden.py
The GPU box never runs this; it only reads the committed golden.npz.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import oracle as orc  # noqa: E402


def ref_fill3(seed, B, H, N, D, bf16=False):
    n = B * H * N * D
    a = orc.ref_fill(seed, 3 * n, bf16=bf16).reshape(3, B, H, N, D)
    return a[0].copy(), a[1].copy(), a[2].copy()


def main():
    if not orc.ref_available():
        subprocess_build()
    out = {}
    # const V (seed 5; Q then K from one stream; V columns = 0.25 * c)
    B, H, N, D = 1, 1, 192, 64
    qk = orc.ref_fill(5, 2 * N * D, bf16=False).reshape(2, B, H, N, D)
    q, k = qk[0].copy(), qk[1].copy()
    v = np.tile((0.25 * np.arange(D, dtype=np.float32))[None, None, None, :], (B, H, N, 1))
    out["const_v.o_kernel"] = orc.ref_attention_fwd(q, k, v, workers=3, bf16=False, threaded=False)
    out["const_v.prefix"] = orc.ref_fill(5, 64, bf16=False)
    # dense d=64 / d=128 (seed 100 + d, N = 384, 3 workers)
    for d in (64, 128):
        q, k, v = ref_fill3(100 + d, 1, 1, 384, d)
        out[f"dense_d{d}.o_kernel"] = orc.ref_attention_fwd(q, k, v, workers=3, bf16=False, threaded=False)
        out[f"dense_d{d}.o_ref_oracle"] = orc.ref_oracle_attention(q[0, 0], k[0, 0], v[0, 0])
        out[f"dense_d{d}.prefix"] = orc.ref_fill(100 + d, 64, bf16=False)
    # KV-chunk invariance (seed 321, N = 384, d = 64)
    q, k, v = ref_fill3(321, 1, 1, 384, 64)
    for kv in (384, 192, 128):
        out[f"chunk_kv{kv}.o_kernel"] = orc.ref_attention_fwd(q, k, v, kv_rows=kv, workers=3, bf16=False,
                                                              threaded=False)
    # B = H = 2 (seed 55, N = 192)
    q, k, v = ref_fill3(55, 2, 2, 192, 64)
    out["bh2.o_kernel"] = orc.ref_attention_fwd(q, k, v, workers=3, bf16=False, threaded=False)
    # BASELINE configs[0]: B1 H8 N1024 D64, bf16-rounded inputs, kv_rows=128, 4 workers
    q, k, v = ref_fill3(0, 1, 8, 1024, 64, bf16=True)
    o = orc.ref_attention_fwd(q, k, v, kv_rows=128, workers=4, bf16=True, threaded=True)
    for hh in (0, 7):
        out[f"c1.h{hh}.o_kernel"] = o[0, hh]
        out[f"c1.h{hh}.o_ref_oracle"] = orc.ref_oracle_attention(q[0, hh], k[0, hh], v[0, hh]).astype(np.float32)
    out["c1.prefix"] = orc.ref_fill(0, 64, bf16=True)
    # the reference's validation verdicts (kernels.hpp:188-202) for the C-ABI tests
    import ctypes
    err = ctypes.create_string_buffer(256)
    L = orc.ref_lib()
    out["validate.c1_stock"] = np.array(L.kref_validate(1, 8, 1024, 64, 0, 0, err, 256))
    out["validate.n200"] = np.array(L.kref_validate(1, 1, 200, 64, 0, 0, err, 256))
    out["validate.d96"] = np.array(L.kref_validate(1, 1, 384, 96, 0, 0, err, 256))
    out["constants.tau"] = np.array([L.kref_temperature_scale(64), L.kref_temperature_scale(128)])
    out["constants.kv_rows"] = np.array([L.kref_kv_tile_rows(64), L.kref_kv_tile_rows(128)])
    # .npy KAT dumps in the reference's own on-disk format (npy.hpp):
    # the dense d=64 case (test_kernels.cpp:128-146), written by the reference's writer
    npy_dir = os.path.join(os.path.dirname(os.path.abspath(__file__)), "npy")
    os.makedirs(npy_dir, exist_ok=True)
    q, k, v = ref_fill3(164, 1, 1, 384, 64)
    for name, arr in (("q", q[0, 0]), ("k", k[0, 0]), ("v", v[0, 0]), ("o_ref", out["dense_d64.o_kernel"][0, 0])):
        orc.ref_save_npy(os.path.join(npy_dir, f"dense_d64_{name}.npy"), arr)
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, os.path.getsize(path), "bytes,", len(out), "arrays")


def subprocess_build():
    import subprocess

    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)


if __name__ == "__main__":
    main()
