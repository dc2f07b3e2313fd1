// tkb_mgpu.cpp — C++ multi-GPU driver for the attention hot path.
//
// One host thread per visible GPU; each thread takes its contiguous share of the
// flattened batch x head grid (tkb_shard_range), allocates its shard, runs forward +
// backward through the C++ host API (include/tkb/attention.hpp -> C ABI) and times it
// with CUDA events. No collective: shards are independent; the host joins the threads
// and reports the max over devices. Optionally (--check) each device verifies head 0 of
// its shard against the CPU oracle (oracle/liboracle.so, loaded at run time).
//
//   tools/tkb_mgpu [--gpus N] [--batch B] [--heads H] [--seq N] [--dim D] [--causal 0|1]
//                  [--iters K] [--check]
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

#define CK(x)                                                                                     \
    do {                                                                                          \
        cudaError_t e_ = (x);                                                                     \
        if (e_ != cudaSuccess) {                                                                  \
            std::fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
            std::exit(2);                                                                         \
        }                                                                                         \
    } while (0)

struct Args {
    int gpus = 0, batch = 16, heads = 16, seq = 4096, dim = 128, causal = 1, iters = 5;
    bool check = false;
};

struct Result {
    double ms = 0;
    int64_t units = 0;
    double max_err = 0;
    std::string err;
};

// splitmix-based uniform(-1, 1) rounded to bf16 (device inputs; per global unit seed so a
// shard equals the same slice of a single-GPU run)
float uni(uint64_t& s) {
    s += 0x9E3779B97F4A7C15ull;
    uint64_t z = s;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    return (float)((z >> 40) * (1.0 / 16777216.0)) * 2.f - 1.f;
}

void run_device(int dev, const Args& a, int world, Result* out) {
    try {
        CK(cudaSetDevice(dev));
        const int64_t units = (int64_t)a.batch * a.heads;
        int64_t u0, u1;
        tkb::shard_range(units, dev, world, u0, u1);
        const int64_t mine = u1 - u0;
        out->units = mine;
        if (mine == 0) return;
        const size_t elems = (size_t)mine * a.seq * a.dim;
        std::vector<__nv_bfloat16> host(elems * 4);
        std::vector<float> hostf(elems * 4);
        for (int t = 0; t < 4; ++t)
            for (int64_t u = 0; u < mine; ++u) {
                uint64_t s = ((uint64_t)(u0 + u) << 8) ^ (uint64_t)t;
                for (size_t i = 0; i < (size_t)a.seq * a.dim; ++i) {
                    const size_t idx = t * elems + (size_t)u * a.seq * a.dim + i;
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
        CK(cudaStreamCreate(&st));
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
        if (a.check) {
            void* h = dlopen("oracle/liboracle.so", RTLD_NOW);
            if (!h) throw tkb::Error("--check needs oracle/liboracle.so (make -C oracle)");
            using Fwd = void (*)(const float*, const float*, const float*, int64_t, int, int, int, double, double*,
                                 double*, int);
            auto fwd = (Fwd)dlsym(h, "tkb_oracle_attn_fwd");
            const size_t hd = (size_t)a.seq * a.dim;
            std::vector<double> ro(hd), rl(a.seq);
            fwd(hostf.data(), hostf.data() + elems, hostf.data() + 2 * elems, 1, a.seq, a.dim, a.causal,
                1.0 / std::sqrt((double)a.dim), ro.data(), rl.data(), 4);
            std::vector<__nv_bfloat16> go(hd);
            CK(cudaMemcpy(go.data(), o, hd * 2, cudaMemcpyDeviceToHost));
            for (size_t i = 0; i < hd; ++i)
                out->max_err = std::max(out->max_err, std::fabs((double)__bfloat162float(go[i]) - ro[i]));
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
        auto nxt = [&] { return std::atoi(argv[++i]); };
        if (s == "--gpus") a.gpus = nxt();
        else if (s == "--batch") a.batch = nxt();
        else if (s == "--heads") a.heads = nxt();
        else if (s == "--seq") a.seq = nxt();
        else if (s == "--dim") a.dim = nxt();
        else if (s == "--causal") a.causal = nxt();
        else if (s == "--iters") a.iters = nxt();
        else if (s == "--check") a.check = true;
    }
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    const int world = a.gpus > 0 ? std::min(a.gpus, ndev) : ndev;
    std::vector<Result> res(world);
    std::vector<std::thread> th;
    for (int d = 0; d < world; ++d) th.emplace_back(run_device, d, std::cref(a), world, &res[d]);
    for (auto& t : th) t.join();
    double ms = 0, err = 0;
    for (int d = 0; d < world; ++d) {
        if (!res[d].err.empty()) {
            std::fprintf(stderr, "device %d: %s\n", d, res[d].err.c_str());
            return 1;
        }
        ms = std::max(ms, res[d].ms);
        err = std::max(err, res[d].max_err);
    }
    const double f = (4.0 + 10.0) * a.batch * a.heads * (double)a.seq * a.seq * a.dim * (a.causal ? 0.5 : 1.0);
    std::printf("{\"gpus\": %d, \"ms_per_step\": %.4f, \"tflops_total\": %.1f, \"tflops_per_gpu\": %.1f%s}\n", world,
                ms, f / (ms / 1e3) / 1e12, f / (ms / 1e3) / 1e12 / world,
                a.check ? (std::string(", \"max_abs_err_head0\": ") + std::to_string(err)).c_str() : "");
    return 0;
}
