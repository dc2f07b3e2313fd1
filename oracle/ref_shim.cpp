// ref_shim.cpp — C-ABI wrapper around the UNMODIFIED reference (kittensim)
// attention path, compiled from the reference headers where they lie
// (/root/reference/proj/include) by oracle/Makefile into oracle/_ref/.
//
// TEST / BASELINE INFRASTRUCTURE ONLY: used to pin the oracle (golden vectors,
// tests/golden/make_golden.py) and as the timed CPU reference arm of bench.py.
// No reference source is copied here; this file only calls its public API:
//   AttentionConfig / AttentionGlobals   kernels.hpp:168-213
//   attention_fwd_kernel                 kernels.hpp:250-343
//   attention_pipeline_config            kernels.hpp:345-355
//   execute_functional (+ExecOptions)    lcsf.hpp:283-289, 779-819
//   oracle_attention                     oracles.hpp:34-64
//   round_to_bf16                        tiles.hpp:40-46
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <random>
#include <string>

#include "kittensim/errors.hpp"
#include "kittensim/kernels.hpp"
#include "kittensim/lcsf.hpp"
#include "kittensim/oracles.hpp"

#define KREF_API extern "C" __attribute__((visibility("default")))

using namespace kittensim;

namespace {
void set_err(char* err, int errlen, const std::string& msg) {
    if (err && errlen > 0) {
        std::strncpy(err, msg.c_str(), (size_t)errlen - 1);
        err[errlen - 1] = 0;
    }
}
int code_of(const std::exception& e) {
    if (dynamic_cast<const ConfigError*>(&e)) return 1;
    if (dynamic_cast<const ShapeError*>(&e)) return 2;
    if (dynamic_cast<const BoundsError*>(&e)) return 3;
    if (dynamic_cast<const ContractViolation*>(&e)) return 6;
    if (dynamic_cast<const DeadlockError*>(&e)) return 7;
    return 9;
}
AttentionConfig make_cfg(int B, int H, int N, int D, int kv_rows, int workers, int bf16) {
    AttentionConfig cfg;
    cfg.batches = B;
    cfg.heads = H;
    cfg.seq = N;
    cfg.head_dim = D;
    cfg.kv_rows = kv_rows;
    if (workers > 0) cfg.num_workers = workers;
    cfg.dtype = bf16 ? Dtype::Bf16 : Dtype::Fp32;
    return cfg;
}
}  // namespace

// AttentionConfig::validate(): 0 ok, else the taxonomy code (1 = ConfigError).
KREF_API int kref_validate(int B, int H, int N, int D, int kv_rows, int workers, char* err, int errlen) {
    try {
        make_cfg(B, H, N, D, kv_rows, workers, 0).validate();
        return 0;
    } catch (const std::exception& e) {
        set_err(err, errlen, e.what());
        return code_of(e);
    }
}

KREF_API int kref_kv_tile_rows(int D) {
    AttentionConfig c;
    c.head_dim = D;
    return c.kv_tile_rows();
}

KREF_API double kref_temperature_scale(int D) {
    AttentionConfig c;
    c.head_dim = D;
    return c.temperature_scale();
}

KREF_API float kref_round_to_bf16(float x) { return round_to_bf16(x); }

// The reference kernel path: execute_functional(attention_fwd_kernel(cfg, g), pipeline).
// q/k/v/o are [B,H,N,D] fp32 (bf16-representable if bf16 = 1). threaded = 1 selects
// the real-thread LCSF backend (lcsf.hpp:595-775), else the seeded interleaver.
KREF_API int kref_attention_fwd(int B, int H, int N, int D, int kv_rows, int workers, int bf16, int threaded,
                                uint64_t seed, const float* q, const float* k, const float* v, float* o, char* err,
                                int errlen) {
    try {
        AttentionConfig cfg = make_cfg(B, H, N, D, kv_rows, workers, bf16);
        auto g = std::make_shared<AttentionGlobals>(cfg);
        const size_t n = (size_t)B * H * N * D;
        std::memcpy(g->q.data.data(), q, n * 4);
        std::memcpy(g->k.data.data(), k, n * 4);
        std::memcpy(g->v.data.data(), v, n * 4);
        ExecOptions opts;
        opts.backend = threaded ? ExecOptions::Backend::Threaded : ExecOptions::Backend::Interleaved;
        opts.seed = seed;
        execute_functional(attention_fwd_kernel(cfg, g), attention_pipeline_config(cfg), opts);
        std::memcpy(o, g->o.data.data(), n * 4);
        return 0;
    } catch (const std::exception& e) {
        set_err(err, errlen, e.what());
        return code_of(e);
    }
}

// The reference fp64 oracle for one head (oracles.hpp:34-64).
KREF_API int kref_oracle_attention(const double* q, const double* k, const double* v, int nq, int nk, int d,
                                   double* out) {
    try {
        std::vector<double> qq(q, q + (size_t)nq * d), kk(k, k + (size_t)nk * d), vv(v, v + (size_t)nk * d);
        auto r = oracle_attention(qq, kk, vv, nq, nk, d);
        std::memcpy(out, r.data(), r.size() * 8);
        return 0;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

// The reference tests' generator: std::mt19937(seed) + uniform_real_distribution<float>(lo, hi),
// round_to_bf16 when bf16 (report.hpp:57-61, test_kernels.cpp:14-18).
KREF_API void kref_fill(uint32_t seed, float lo, float hi, int bf16, float* out, int64_t total) {
    std::mt19937 rng(seed);
    std::uniform_real_distribution<float> u(lo, hi);
    for (int64_t i = 0; i < total; ++i) out[i] = bf16 ? round_to_bf16(u(rng)) : u(rng);
}

// The reference fp64 rotary oracle (oracles.hpp:66-90) for one [n x hd] head.
KREF_API int kref_oracle_rotary(const double* x, const double* sin_tab, const double* cos_tab, int n, int hd,
                                double* out) {
    try {
        std::vector<double> xx(x, x + (size_t)n * hd), ss(sin_tab, sin_tab + (size_t)n * hd / 2),
            cc(cos_tab, cos_tab + (size_t)n * hd / 2);
        auto r = oracle_rotary(xx, ss, cc, n, hd);
        std::memcpy(out, r.data(), r.size() * 8);
        return 0;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

// The reference rotary kernel (kernels.hpp:413-503) through execute_functional, fp32.
KREF_API int kref_rotary(int B, int H, int N, int hd, int workers, const float* x, const float* sin_tab,
                         const float* cos_tab, float* o, char* err, int errlen) {
    try {
        RotaryConfig cfg;
        cfg.batches = B;
        cfg.heads = H;
        cfg.seq = N;
        cfg.head_dim = hd;
        cfg.num_workers = workers;
        auto g = std::make_shared<RotaryGlobals>(cfg);
        std::memcpy(g->x.data.data(), x, (size_t)B * H * N * hd * 4);
        std::memcpy(g->sin_tab.data.data(), sin_tab, (size_t)N * hd / 2 * 4);
        std::memcpy(g->cos_tab.data.data(), cos_tab, (size_t)N * hd / 2 * 4);
        execute_functional(rotary_kernel(cfg, g), rotary_pipeline_config(cfg));
        std::memcpy(o, g->o.data.data(), (size_t)B * H * N * hd * 4);
        return 0;
    } catch (const std::exception& e) {
        set_err(err, errlen, e.what());
        return code_of(e);
    }
}

// The reference fp64 GEMM oracle (oracles.hpp:17-30).
KREF_API int kref_oracle_gemm(const double* a, const double* b, int m, int n, int k, double* c) {
    try {
        std::vector<double> aa(a, a + (size_t)m * k), bb(b, b + (size_t)k * n);
        auto r = oracle_gemm(aa, bb, m, n, k);
        std::memcpy(c, r.data(), r.size() * 8);
        return 0;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

// The reference GEMM kernel (kernels.hpp:76-149) through execute_functional (fp32 or emulated bf16).
KREF_API int kref_gemm(int m, int n, int k, int m_block, int n_block, int super_m, int bf16, const float* a,
                       const float* b, float* c, char* err, int errlen) {
    try {
        GemmConfig cfg;
        cfg.m = m;
        cfg.n = n;
        cfg.k = k;
        cfg.m_block = m_block;
        cfg.n_block = n_block;
        cfg.super_m = super_m;
        cfg.dtype = bf16 ? Dtype::Bf16 : Dtype::Fp32;
        auto g = std::make_shared<GemmGlobals>(cfg);
        std::memcpy(g->a.data.data(), a, (size_t)m * k * 4);
        std::memcpy(g->b.data.data(), b, (size_t)k * n * 4);
        execute_functional(gemm_kernel(cfg, g), gemm_pipeline_config(cfg));
        std::memcpy(c, g->c.data.data(), (size_t)m * n * 4);
        return 0;
    } catch (const std::exception& e) {
        set_err(err, errlen, e.what());
        return code_of(e);
    }
}

// supergroup_order (grid.hpp:28-47): the reference launch order, as (row, col) pairs.
KREF_API int kref_supergroup_order(int r_blocks, int c_blocks, int super_m, int* rows, int* cols) {
    try {
        auto o = supergroup_order(r_blocks, c_blocks, super_m);
        for (size_t i = 0; i < o.size(); ++i) {
            rows[i] = o[i].row;
            cols[i] = o[i].col;
        }
        return 0;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

