// tkb/attention.hpp — C++ host mirror of the reference's attention interface over the
// C ABI (include/tkb_attn.h). Header-only; link libtkb.so.
//
// Reference (kittensim, /root/reference/proj/include/kittensim):
//   struct AttentionConfig { batches, heads, seq, head_dim, ... }   kernels.hpp:168-203
//   AttentionConfig::validate()  -> throws ConfigError                kernels.hpp:188-202
//   temperature_scale()          -> tau = d^-1/2 * log2(e)            kernels.hpp:184-186
//   struct AttentionGlobals { GlobalTensor q, k, v, o; }             kernels.hpp:205-213
//   execute_functional(attention_fwd_kernel(cfg, g), pipeline_cfg)   kernels.hpp:250-355
//   exceptions Error/ConfigError/ShapeError/BoundsError/...          errors.hpp:9-46
//
// Here the globals are device pointers, the call is asynchronous on a CUDA stream, and
// the CPU-model knobs (kv_rows, qo_rows, num_workers, dtype) are compile-time kernel
// choices. New: causal, the saved L, and the backward.
#pragma once
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <stdexcept>
#include <string>

#include "../tkb_attn.h"

namespace tkb {

struct Error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct ConfigError : Error {
    using Error::Error;
};
struct ShapeError : Error {
    using Error::Error;
};
struct BoundsError : Error {
    using Error::Error;
};
struct ContractViolation : Error {
    using Error::Error;
};
struct UnsupportedDevice : Error {
    using Error::Error;
};
struct CudaError : Error {
    using Error::Error;
};

inline void check(int rc) {
    if (rc == TKB_OK) return;
    const std::string msg = tkb_last_error();
    switch (rc) {
        case TKB_ERR_CONFIG: throw ConfigError(msg);
        case TKB_ERR_SHAPE: throw ShapeError(msg);
        case TKB_ERR_BOUNDS: throw BoundsError(msg);
        case TKB_ERR_UNSUPPORTED: throw UnsupportedDevice(msg);
        case TKB_ERR_CUDA: throw CudaError(msg);
        case TKB_ERR_CONTRACT: throw ContractViolation(msg);
        default: throw Error(msg);
    }
}

struct AttentionConfig {
    int batches = 1;
    int heads = 1;
    int seq = 0;
    int head_dim = 0;  // 64 or 128
    bool causal = false;
    float softmax_scale = 0.f;  // 0: head_dim^-1/2
    bool check_finite = false;  // kernels.hpp:277-284, opt-in (synchronises the stream)
    int kv_heads = 0;           // grouped-query attention: 0 = heads, else heads % kv_heads == 0

    double temperature_scale() const {
        const double s = softmax_scale > 0.f ? softmax_scale : 1.0 / std::sqrt((double)head_dim);
        return s * 1.44269504089;
    }
    tkb_attn_desc desc() const {
        tkb_attn_desc d;
        tkb_attn_desc_init(&d, batches, heads, seq, head_dim, causal ? 1 : 0);
        d.softmax_scale = softmax_scale;
        d.check_finite = check_finite ? 1 : 0;
        d.kv_heads = kv_heads;
        return d;
    }
    void validate() const {
        const tkb_attn_desc d = desc();
        check(tkb_attn_validate(&d));
    }
};

// Device pointers, [B, H, N, D] bf16 contiguous; lse fp32 [B, H, N].
struct AttentionGlobals {
    const void* q = nullptr;
    const void* k = nullptr;
    const void* v = nullptr;
    void* o = nullptr;
    float* lse = nullptr;
};

struct AttentionGrads {
    const void* dout = nullptr;
    void* dq = nullptr;
    void* dk = nullptr;
    void* dv = nullptr;
};

// Forward: the attention_fwd_kernel + execute_functional pair of the reference.
inline void attention_fwd(const AttentionConfig& cfg, const AttentionGlobals& g, void* cuda_stream = nullptr) {
    const tkb_attn_desc d = cfg.desc();
    check(tkb_attn_fwd(&d, g.q, g.k, g.v, g.o, g.lse, cuda_stream));
}

inline std::size_t attention_bwd_workspace_bytes(const AttentionConfig& cfg) {
    const tkb_attn_desc d = cfg.desc();
    return tkb_attn_bwd_workspace_bytes(&d);
}

// Backward from the saved L (new; deterministic).
inline void attention_bwd(const AttentionConfig& cfg, const AttentionGlobals& g, const AttentionGrads& gr,
                          void* workspace, std::size_t workspace_bytes, void* cuda_stream = nullptr) {
    const tkb_attn_desc d = cfg.desc();
    check(tkb_attn_bwd(&d, g.q, g.k, g.v, g.o, gr.dout, g.lse, gr.dq, gr.dk, gr.dv, workspace, workspace_bytes,
                       cuda_stream));
}

// Variable-length batches (tkb_attn_fwd_varlen / tkb_attn_bwd_varlen): cfg.batches sequences,
// cfg.seq = the longest; tensors packed token-major [T, H, D] / [T, Hkv, D], contiguous;
// cu_seqlens is a device int32 [batches + 1]; lse fp32 [batches, heads, seq]. Workspaces are
// caller-owned device buffers (128-byte aligned) of the *_workspace_bytes sizes.
inline std::size_t attention_fwd_varlen_workspace_bytes(const AttentionConfig& cfg) {
    const tkb_attn_desc d = cfg.desc();
    return tkb_attn_fwd_varlen_workspace_bytes(&d);
}
inline std::size_t attention_bwd_varlen_workspace_bytes(const AttentionConfig& cfg) {
    const tkb_attn_desc d = cfg.desc();
    return tkb_attn_bwd_varlen_workspace_bytes(&d);
}
inline void attention_fwd_varlen(const AttentionConfig& cfg, const int32_t* cu_seqlens, int64_t total_tokens,
                                 const AttentionGlobals& g, void* workspace, std::size_t workspace_bytes,
                                 void* cuda_stream = nullptr) {
    const tkb_attn_desc d = cfg.desc();
    check(tkb_attn_fwd_varlen(&d, cu_seqlens, total_tokens, g.q, g.k, g.v, g.o, g.lse, workspace, workspace_bytes,
                              cuda_stream));
}
inline void attention_bwd_varlen(const AttentionConfig& cfg, const int32_t* cu_seqlens, int64_t total_tokens,
                                 const AttentionGlobals& g, const AttentionGrads& gr, void* workspace,
                                 std::size_t workspace_bytes, void* cuda_stream = nullptr) {
    const tkb_attn_desc d = cfg.desc();
    check(tkb_attn_bwd_varlen(&d, cu_seqlens, total_tokens, g.q, g.k, g.v, g.o, gr.dout, g.lse, gr.dq, gr.dk,
                              gr.dv, workspace, workspace_bytes, cuda_stream));
}

// D = 128 backward dK/dV on 2-CTA clusters (tcgen05 cta_group::2); calling thread only, default off.
inline void set_bwd_pairs(bool on) { check(tkb_set_bwd_pairs(on ? 1 : 0)); }

// Multi-GPU driver helper: this rank's contiguous share of the batch x head grid.
inline void shard_range(int64_t units, int rank, int world, int64_t& begin, int64_t& end) {
    check(tkb_shard_range(units, rank, world, &begin, &end));
}

}  // namespace tkb
