// tkb_mgpu.cpp — C++ multi-GPU driver for the attention hot path.
//
// One host thread per rank; rank r runs on visible device r % ndev (so --world 2 on a
// single GPU runs two ranks side by side on it, each on its own stream). Each rank takes
// its contiguous share of the flattened batch x head grid (tkb_shard_range), generates its
// shard from per-(global unit) seeds, runs forward + backward through the C++ host API
// (include/tkb/attention.hpp -> C ABI) and times it with CUDA events. No collective:
// shards are independent; the host joins the threads and reports the max over ranks.
//
//   --check   each rank verifies the first head of its shard (O, L, dQ, dK, dV) against
//             the CPU oracle (oracle/liboracle.so, dlopen'ed at run time — test only)
//   --hashes  prints a 64-bit FNV-1a hash of every unit's O, L, dQ, dK, dV bytes, so a
//             sharded run can be compared bit for bit with a single-rank run
//
//   tools/tkb_mgpu [--world W] [--batch B] [--heads H] [--seq N] [--dim D] [--causal 0|1]
//                  [--iters K] [--check] [--hashes]
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../include/tkb/attention.hpp"

namespace {

#define CK(x)                                                                                         \
    do {                                                                                              \
        cudaError_t e_ = (x);                                                                         \
        if (e_ != cudaSuccess)                                                                        \
            throw tkb::CudaError(std::string(#x) + ": " + cudaGetErrorString(e_));                    \
    } while (0)

struct Args {
    int world = 0, batch = 16, heads = 16, seq = 4096, dim = 128, causal = 1, iters = 5;
    bool check = false, hashes = false;
};

struct Result {
    double ms = 0;
    int64_t u0 = 0, units = 0;
    double err_o = 0, err_l = 0, err_dq = 0, err_dk = 0, err_dv = 0;
    std::vector<unsigned long long> hashes;
    std::string err;
};

// splitmix-based uniform(-1, 1) (device inputs; per global unit seed so a shard equals the
// same slice of a single-rank run)
float uni(uint64_t& s) {
    s += 0x9E3779B97F4A7C15ull;
    uint64_t z = s;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    return (float)((z >> 40) * (1.0 / 16777216.0)) * 2.f - 1.f;
}

unsigned long long fnv(const void* p, size_t n, unsigned long long h) {
    const unsigned char* b = static_cast<const unsigned char*>(p);
    for (size_t i = 0; i < n; ++i) h = (h ^ b[i]) * 1099511628211ull;
    return h;
}

double max_abs(const __nv_bfloat16* got, const double* ref, size_t n) {
    double m = 0;
    for (size_t i = 0; i < n; ++i) m = std::max(m, std::fabs((double)__bfloat162float(got[i]) - ref[i]));
    return m;
}

void run_rank(int rank, int dev, const Args& a, int world, Result* out) {
    try {
        CK(cudaSetDevice(dev));
        const int64_t units = (int64_t)a.batch * a.heads;
        int64_t u0, u1;
        tkb::shard_range(units, rank, world, u0, u1);
        const int64_t mine = u1 - u0;
        out->u0 = u0;
        out->units = mine;
        if (mine == 0) return;
        const size_t hd = (size_t)a.seq * a.dim;
        const size_t elems = (size_t)mine * hd;
        std::vector<__nv_bfloat16> host(elems * 4);
        std::vector<float> hostf(elems * 4);
        for (int t = 0; t < 4; ++t)  // q, k, v, dO
            for (int64_t u = 0; u < mine; ++u) {
                uint64_t s = ((uint64_t)(u0 + u) << 8) ^ (uint64_t)t;
                for (size_t i = 0; i < hd; ++i) {
                    const size_t idx = t * elems + (size_t)u * hd + i;
                    host[idx] = __float2bfloat16(uni(s));
                    hostf[idx] = __bfloat162float(host[idx]);
                }
            }
        __nv_bfloat16 *q, *k, *v, *o, *dO, *dq, *dk, *dv;
        float* lse;
        void* ws;
        CK(cudaMalloc(&q, elems * 2 * 8));
        k = q + elems;
        v = k + elems;
        dO = v + elems;
        o = dO + elems;
        dq = o + elems;
        dk = dq + elems;
        dv = dk + elems;
        CK(cudaMalloc(&lse, (size_t)mine * a.seq * 4));
        CK(cudaMemcpy(q, host.data(), elems * 2 * 4, cudaMemcpyHostToDevice));
        tkb::AttentionConfig cfg;
        cfg.batches = 1;
        cfg.heads = (int)mine;
        cfg.seq = a.seq;
        cfg.head_dim = a.dim;
        cfg.causal = a.causal != 0;
        cfg.validate();
        const size_t wsb = tkb::attention_bwd_workspace_bytes(cfg);
        CK(cudaMalloc(&ws, wsb));
        cudaStream_t st;
        CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        tkb::AttentionGlobals g{q, k, v, o, lse};
        tkb::AttentionGrads gr{dO, dq, dk, dv};
        auto step = [&] {
            tkb::attention_fwd(cfg, g, st);
            tkb::attention_bwd(cfg, g, gr, ws, wsb, st);
        };
        for (int i = 0; i < 3; ++i) step();
        cudaEvent_t e0, e1;
        CK(cudaEventCreate(&e0));
        CK(cudaEventCreate(&e1));
        CK(cudaStreamSynchronize(st));
        CK(cudaEventRecord(e0, st));
        for (int i = 0; i < a.iters; ++i) step();
        CK(cudaEventRecord(e1, st));
        CK(cudaEventSynchronize(e1));
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        out->ms = ms / a.iters;
        if (a.hashes || a.check) {
            std::vector<__nv_bfloat16> res(elems * 4);  // o, dq, dk, dv
            std::vector<float> rl((size_t)mine * a.seq);
            CK(cudaMemcpy(res.data(), o, elems * 2 * 4, cudaMemcpyDeviceToHost));
            CK(cudaMemcpy(rl.data(), lse, rl.size() * 4, cudaMemcpyDeviceToHost));
            if (a.hashes)
                for (int64_t u = 0; u < mine; ++u) {
                    unsigned long long h = 1469598103934665603ull;
                    for (int t = 0; t < 4; ++t) h = fnv(res.data() + t * elems + (size_t)u * hd, hd * 2, h);
                    h = fnv(rl.data() + (size_t)u * a.seq, (size_t)a.seq * 4, h);
                    out->hashes.push_back(h);
                }
            if (a.check) {
                void* h = dlopen("oracle/liboracle.so", RTLD_NOW);
                if (!h) throw tkb::Error("--check needs oracle/liboracle.so (make -C oracle)");
                using Fwd = void (*)(const float*, const float*, const float*, int64_t, int, int, int, double,
                                     double*, double*, int);
                using Bwd = void (*)(const float*, const float*, const float*, const float*, int64_t, int, int, int,
                                     double, double*, double*, double*, int);
                auto fwd = (Fwd)dlsym(h, "tkb_oracle_attn_fwd");
                auto bwd = (Bwd)dlsym(h, "tkb_oracle_attn_bwd");
                if (!fwd || !bwd) throw tkb::Error("oracle symbols missing");
                const double scale = 1.0 / std::sqrt((double)a.dim);
                std::vector<double> ro(hd), rlse(a.seq), rdq(hd), rdk(hd), rdv(hd);
                const float *hq = hostf.data(), *hk = hq + elems, *hv = hk + elems, *hdo = hv + elems;
                fwd(hq, hk, hv, 1, a.seq, a.dim, a.causal, scale, ro.data(), rlse.data(), 4);
                bwd(hq, hk, hv, hdo, 1, a.seq, a.dim, a.causal, scale, rdq.data(), rdk.data(), rdv.data(), 4);
                out->err_o = max_abs(res.data(), ro.data(), hd);
                out->err_dq = max_abs(res.data() + elems, rdq.data(), hd);
                out->err_dk = max_abs(res.data() + 2 * elems, rdk.data(), hd);
                out->err_dv = max_abs(res.data() + 3 * elems, rdv.data(), hd);
                for (int i = 0; i < a.seq; ++i) out->err_l = std::max(out->err_l, std::fabs(rl[i] - rlse[i]));
            }
        }
        cudaFree(q);
        cudaFree(lse);
        cudaFree(ws);
        cudaStreamDestroy(st);
    } catch (const std::exception& e) {
        out->err = e.what();
    }
}

}  // namespace

int main(int argc, char** argv) {
    Args a;
    for (int i = 1; i < argc; ++i) {
        std::string s = argv[i];
        auto nxt = [&] { return i + 1 < argc ? std::atoi(argv[++i]) : 0; };
        if (s == "--world" || s == "--gpus") a.world = nxt();
        else if (s == "--batch") a.batch = nxt();
        else if (s == "--heads") a.heads = nxt();
        else if (s == "--seq") a.seq = nxt();
        else if (s == "--dim") a.dim = nxt();
        else if (s == "--causal") a.causal = nxt();
        else if (s == "--iters") a.iters = nxt();
        else if (s == "--check") a.check = true;
        else if (s == "--hashes") a.hashes = true;
    }
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1) {
        std::fprintf(stderr, "no CUDA device\n");
        return 2;
    }
    const int world = a.world > 0 ? a.world : ndev;
    std::vector<Result> res(world);
    std::vector<std::thread> th;
    for (int r = 0; r < world; ++r) th.emplace_back(run_rank, r, r % ndev, std::cref(a), world, &res[r]);
    for (auto& t : th) t.join();
    double ms = 0, eo = 0, el = 0, edq = 0, edk = 0, edv = 0;
    for (int r = 0; r < world; ++r) {
        if (!res[r].err.empty()) {
            std::fprintf(stderr, "rank %d: %s\n", r, res[r].err.c_str());
            return 1;
        }
        ms = std::max(ms, res[r].ms);
        eo = std::max(eo, res[r].err_o);
        el = std::max(el, res[r].err_l);
        edq = std::max(edq, res[r].err_dq);
        edk = std::max(edk, res[r].err_dk);
        edv = std::max(edv, res[r].err_dv);
    }
    const double f = (4.0 + 10.0) * a.batch * a.heads * (double)a.seq * a.seq * a.dim * (a.causal ? 0.5 : 1.0);
    std::string extra;
    if (a.check) {
        char buf[256];
        std::snprintf(buf, sizeof buf,
                      ", \"max_abs_err\": {\"o\": %.4g, \"lse\": %.4g, \"dq\": %.4g, \"dk\": %.4g, \"dv\": %.4g}", eo,
                      el, edq, edk, edv);
        extra += buf;
    }
    if (a.hashes) {
        extra += ", \"unit_hashes\": [";
        bool first = true;
        for (int r = 0; r < world; ++r)
            for (unsigned long long h : res[r].hashes) {
                extra += (first ? "\"" : ", \"") + std::to_string(h) + "\"";
                first = false;
            }
        extra += "]";
    }
    std::printf("{\"ranks\": %d, \"devices\": %d, \"ms_per_step\": %.4f, \"tflops_total\": %.1f, "
                "\"tflops_per_rank\": %.1f%s}\n",
                world, std::min(world, ndev), ms, f / (ms / 1e3) / 1e12, f / (ms / 1e3) / 1e12 / world,
                extra.c_str());
    return 0;
}
