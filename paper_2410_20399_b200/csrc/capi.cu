// capi.cu — the C-ABI boundary (include/tkb_attn.h): validation with the
// reference's error taxonomy, TMA descriptor construction, launches.
// Never throws across the ABI; the last error message is thread-local.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <atomic>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "attn_common.cuh"
#include "host/tmap.hpp"
#include "tkb_attn.h"

namespace tkb {
int launch_attn_bwd(int head_dim, bool causal, const BwdParams& p, int batches, const void* o, const void* dout,
                    const float* lse, float* lse2, float* delta, int64_t sb, int64_t sh, int64_t sn,
                    cudaStream_t stream, int phases, int* launches);
int launch_check_finite(const void* const* ptrs, int nptrs, int batches, int heads, int n, int d, int64_t sb,
                        int64_t sh, int64_t sn, int* flag_dev, cudaStream_t stream);
}  // namespace tkb

namespace {

thread_local std::string g_err;
thread_local int g_launches = 0;
// Debug / selection knobs: per host thread, so a profiling thread cannot change what the
// calls of another thread compute (tkb_debug_set_*, tkb_set_bwd_pairs).
thread_local long long* g_trace = nullptr;  // debug timeline (tkb_debug_set_trace)
thread_local int g_trace_every = 1, g_trace_slots = 0;
thread_local int g_bwd_phases = 7;  // debug: bit 0 prep, bit 1 dK/dV kernel, bit 2 dQ kernel
thread_local int g_bwd_pairs = 0;   // D = 128 dK/dV on CTA pairs (tkb_set_bwd_pairs)
thread_local int g_fwd_task_tiles = 0;  // debug: forward query tiles per task (0 = by problem size)

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

// ---------------------------------------------------------------- per-device state
// The persistent attention kernels claim tasks from a device counter pair {claims, CTAs
// done} that the last CTA of the grid resets to zero (lcsf::queue_exit). Two kernels that
// run concurrently must not share a pair, so each (device, stream) gets its own slot of a
// pool allocated once per device (tkb_device_init, or lazily on the first call); kernels on
// one stream are ordered, so they may share its slot. Slot = 4 ints: the counter pair and
// the check_finite flag. Streams are told apart by cudaStreamGetId (unique for the life of
// the process; the per-thread default stream has its own id). When more than kSlots
// streams have been seen, the least recently used slot is recycled.
constexpr int kMaxDevices = 64;
constexpr int kSlots = 4096;

struct DeviceState {
    std::once_flag once;
    int rc = TKB_OK;
    std::string err;
    int sms = 0;
    int* pool = nullptr;  // kSlots x 4 ints, zeroed
    std::mutex mu;
    std::unordered_map<unsigned long long, int> slot_of;  // stream id -> slot
    std::vector<unsigned long long> owner;                // slot -> stream id
    std::vector<unsigned long long> last_use;             // slot -> tick
    unsigned long long tick = 0;
};
DeviceState g_dev[kMaxDevices];

int device_init(int dev) {
    if (dev < 0 || dev >= kMaxDevices) return fail(TKB_ERR_UNSUPPORTED, "device ordinal too large");
    DeviceState& ds = g_dev[dev];
    std::call_once(ds.once, [&] {
        int prev = -1;
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
        cudaDeviceGetAttribute(&ds.sms, cudaDevAttrMultiProcessorCount, dev);
        cudaError_t e = cudaMalloc(&ds.pool, (size_t)kSlots * 4 * sizeof(int));
        if (e == cudaSuccess) e = cudaMemset(ds.pool, 0, (size_t)kSlots * 4 * sizeof(int));
        if (e == cudaSuccess) e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            ds.rc = TKB_ERR_CUDA;
            ds.err = std::string("device state init: ") + cudaGetErrorString(e);
        }
        ds.owner.assign(kSlots, ~0ull);
        ds.last_use.assign(kSlots, 0);
        if (prev >= 0 && prev != dev) cudaSetDevice(prev);
    });
    if (ds.rc != TKB_OK) return fail(ds.rc, ds.err);
    return TKB_OK;
}

// SM count and this stream's slot on the current device.
int device_state(cudaStream_t st, int* sms, int** slot) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return fail(TKB_ERR_CUDA, std::string("cudaGetDevice: ") + cudaGetErrorString(e));
    if (int rc = device_init(dev)) return rc;
    DeviceState& ds = g_dev[dev];
    *sms = ds.sms;
    if (slot == nullptr) return TKB_OK;
    // The slot key: the stream's id, or — while the stream is being captured into a CUDA graph,
    // where cudaStreamGetId is not permitted — the capture's unique id (top bit set). A graph's
    // kernels then own that slot for the graph's lifetime (never recycled), and the graph must
    // not be replayed concurrently with itself.
    unsigned long long id = 0;
    bool captured = false;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    unsigned long long cap_id = 0;
    e = cudaStreamGetCaptureInfo(st, &cs, &cap_id);
    if (e != cudaSuccess) return fail(TKB_ERR_CUDA, std::string("cudaStreamGetCaptureInfo: ") + cudaGetErrorString(e));
    if (cs == cudaStreamCaptureStatusActive) {
        id = (1ull << 63) | cap_id;
        captured = true;
    } else {
        e = cudaStreamGetId(st, &id);
        if (e != cudaSuccess) return fail(TKB_ERR_CUDA, std::string("cudaStreamGetId: ") + cudaGetErrorString(e));
    }
    std::lock_guard<std::mutex> lock(ds.mu);
    int s;
    auto it = ds.slot_of.find(id);
    if (it != ds.slot_of.end()) {
        s = it->second;
    } else if (ds.slot_of.size() < (size_t)kSlots) {
        s = (int)ds.slot_of.size();
        ds.slot_of.emplace(id, s);
        ds.owner[s] = id;
    } else {  // recycle the least recently used slot (never one a captured graph owns)
        s = -1;
        for (int i = 0; i < kSlots; ++i)
            if (ds.last_use[i] != ~0ull && (s < 0 || ds.last_use[i] < ds.last_use[s])) s = i;
        if (s < 0) return fail(TKB_ERR_CONTRACT, "scheduler slots exhausted by captured graphs");
        ds.slot_of.erase(ds.owner[s]);
        ds.slot_of.emplace(id, s);
        ds.owner[s] = id;
    }
    ds.last_use[s] = captured ? ~0ull : ++ds.tick;
    *slot = ds.pool + 4 * s;
    return TKB_OK;
}

// ---------------------------------------------------------------- TMA descriptor cache
// CUtensorMap encoding is a pure function of (base, dims, strides, box, swizzle); a call
// re-encodes 4 (forward) or 9 (backward) maps, so each host thread keeps the most recent
// ones (4-way set-associative on a hash of the key, LRU within a set).
struct MapKey {
    const void* base;
    uint64_t dims[4];
    uint64_t strides[4];
    uint32_t box_rows;
    bool operator==(const MapKey& o) const {
        return base == o.base && box_rows == o.box_rows && std::memcmp(dims, o.dims, sizeof(dims)) == 0 &&
               std::memcmp(strides, o.strides, sizeof(strides)) == 0;
    }
};
struct MapEntry {
    bool valid = false;
    unsigned long long used = 0;  // LRU tick
    MapKey key;
    CUtensorMap map;
};
constexpr int kMapSets = 32, kMapWays = 4;  // 4-way set-associative, LRU within a set
thread_local MapEntry g_maps[kMapSets][kMapWays];
thread_local unsigned long long g_map_hits = 0, g_map_misses = 0, g_map_tick = 0;

uint64_t mix64(uint64_t z) {  // splitmix64 finaliser: every input bit reaches the low bits
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

size_t map_hash(const MapKey& k) {
    uint64_t h = mix64((uint64_t)(uintptr_t)k.base ^ ((uint64_t)k.box_rows << 48));
    for (int i = 0; i < 4; ++i) h = mix64(h ^ k.dims[i] ^ (k.strides[i] << 24));
    return (size_t)h;
}

struct Strides {
    int64_t b, h, n;
};

Strides strides_of(const tkb_attn_desc* d) {
    Strides s;
    s.n = d->stride_n ? d->stride_n : d->head_dim;
    s.h = d->stride_h ? d->stride_h : (int64_t)d->seq * s.n;
    s.b = d->stride_b ? d->stride_b : (int64_t)d->heads * s.h;
    return s;
}

int kv_heads_of(const tkb_attn_desc* d) { return d->kv_heads > 0 ? d->kv_heads : d->heads; }

// strides of k/v/dk/dv ([B, Hkv, N, D]); q's strides when multi-head and none given
Strides kv_strides_of(const tkb_attn_desc* d) {
    if (d->kv_stride_b == 0 && d->kv_stride_h == 0 && d->kv_stride_n == 0 && kv_heads_of(d) == d->heads)
        return strides_of(d);
    Strides s;
    s.n = d->kv_stride_n ? d->kv_stride_n : d->head_dim;
    s.h = d->kv_stride_h ? d->kv_stride_h : (int64_t)d->seq * s.n;
    s.b = d->kv_stride_b ? d->kv_stride_b : (int64_t)kv_heads_of(d) * s.h;
    return s;
}

// Variable-length batches: packed token-major [T, H, D] (q/o/do/dq) and [T, Hkv, D]
// (k/v/dk/dv); stride_n / stride_h are the token / head strides (0 = H D / D), stride_b unused.
struct Varlen {
    const int32_t* cu;  // device [B + 1]
    int64_t total;      // T = cu[B]
};

Strides varlen_strides(const tkb_attn_desc* d, bool kv) {
    const int heads = kv ? kv_heads_of(d) : d->heads;
    const int64_t sn = kv ? d->kv_stride_n : d->stride_n, sh = kv ? d->kv_stride_h : d->stride_h;
    Strides s;
    s.h = sh ? sh : d->head_dim;
    s.n = sn ? sn : (int64_t)heads * d->head_dim;
    s.b = 0;
    return s;
}

float scale_of(const tkb_attn_desc* d) {
    return d->softmax_scale > 0.f ? d->softmax_scale : (float)(1.0 / std::sqrt((double)d->head_dim));
}

int check_device() {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return fail(TKB_ERR_CUDA, std::string("cudaGetDevice: ") + cudaGetErrorString(e));
    static thread_local int cached_dev = -1, cached_ok = 0;
    if (cached_dev != dev) {
        int major = 0, minor = 0;
        cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
        cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
        cached_dev = dev;
        cached_ok = (major == 10 && minor == 0);
        if (!cached_ok)
            return fail(TKB_ERR_UNSUPPORTED, "device compute capability " + std::to_string(major) + "." +
                                                 std::to_string(minor) + " is not sm_100 (B200)");
    }
    return cached_ok ? TKB_OK : fail(TKB_ERR_UNSUPPORTED, "device is not sm_100 (B200)");
}

// 4-D {D, N, H, B} bf16 map with a {64, box_rows, 1, 1} SW128 box (heads = H, or Hkv for k/v),
// through the per-thread descriptor cache.
int make_bhnd_map(CUtensorMap* tm, const void* base, const tkb_attn_desc* d, const Strides& s, int heads = 0,
                  uint32_t box_rows = 128) {
    MapKey key;
    key.base = base;
    key.dims[0] = (uint64_t)d->head_dim;
    key.dims[1] = (uint64_t)d->seq;
    key.dims[2] = (uint64_t)(heads > 0 ? heads : d->heads);
    key.dims[3] = (uint64_t)d->batches;
    key.strides[0] = 1;
    key.strides[1] = (uint64_t)s.n;
    key.strides[2] = (uint64_t)s.h;
    key.strides[3] = (uint64_t)s.b;
    key.box_rows = box_rows;
    MapEntry* set = g_maps[map_hash(key) % kMapSets];
    MapEntry* victim = &set[0];
    for (int w = 0; w < kMapWays; ++w) {
        MapEntry& e = set[w];
        if (e.valid && e.key == key) {
            ++g_map_hits;
            e.used = ++g_map_tick;
            *tm = e.map;
            return TKB_OK;
        }
        if (!e.valid || e.used < victim->used) victim = &e;
    }
    ++g_map_misses;
    uint32_t box[4] = {64, box_rows, 1, 1};
    std::string err;
    if (!tkb::host::make_tmap(tm, base, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, 4, key.dims, key.strides, box,
                              CU_TENSOR_MAP_SWIZZLE_128B, &err))
        return fail(TKB_ERR_SHAPE, "tensor map: " + err);
    victim->valid = true;
    victim->used = ++g_map_tick;
    victim->key = key;
    victim->map = *tm;
    return TKB_OK;
}

// Variable-length batches: the template of one packed tensor ([T, heads, D], strides s) is the
// map of a single sequence of the maximum length at the tensor's base ({D, n_max, heads, 1});
// varlen_maps_kernel copies it per sequence, re-pointed at cu[b] with n_b rows.
int varlen_template(tkb::VarlenMapTemplates* t, int m, const void* base, const tkb_attn_desc* d, const Strides& s,
                    int heads) {
    tkb_attn_desc d1 = *d;
    d1.batches = 1;
    Strides s1 = s;
    s1.b = s.n * d->seq;
    if (int rc = make_bhnd_map(&t->tmpl[m], base, &d1, s1, heads)) return rc;
    t->base[m] = (unsigned long long)(uintptr_t)base;
    t->row_bytes[m] = s.n * 2;
    return TKB_OK;
}

int varlen_maps(tkb::VarlenMapTemplates& t, const Varlen& vl, int batches, void* out, cudaStream_t st) {
    const int e = tkb::launch_varlen_maps(t, vl.cu, batches, reinterpret_cast<CUtensorMap*>(out), st);
    if (e) return fail(TKB_ERR_CUDA, std::string("varlen maps launch: ") + cudaGetErrorString((cudaError_t)e));
    return TKB_OK;
}

size_t round256(size_t b) { return (b + 255) & ~(size_t)255; }
size_t varlen_map_bytes(const tkb_attn_desc* d, int nmaps) { return (size_t)d->batches * nmaps * sizeof(CUtensorMap); }

// The reference's non-finite input scan (kernels.hpp:277-284), opt-in: the flag lives in
// this stream's state slot (no allocation); the result is read back synchronously.
int finite_check(const tkb_attn_desc* d, const void* const* ptrs, int nptrs, const Strides& s, int heads,
                 int* slot, cudaStream_t st, const Varlen* vl = nullptr) {
    int* flag = slot + 2;
    cudaError_t e = cudaMemsetAsync(flag, 0, sizeof(int), st);
    if (e != cudaSuccess) return fail(TKB_ERR_CUDA, std::string("check_finite: ") + cudaGetErrorString(e));
    int rc = vl ? tkb::launch_check_finite(ptrs, nptrs, 1, heads, (int)vl->total, d->head_dim, 0, s.h, s.n, flag, st)
                : tkb::launch_check_finite(ptrs, nptrs, d->batches, heads, d->seq, d->head_dim, s.b, s.h, s.n, flag, st);
    int host = 0;
    e = cudaMemcpyAsync(&host, flag, sizeof(int), cudaMemcpyDeviceToHost, st);
    cudaError_t e2 = cudaStreamSynchronize(st);
    if (rc != 0 || e != cudaSuccess || e2 != cudaSuccess) return fail(TKB_ERR_CUDA, "check_finite launch failed");
    if (host) return fail(TKB_ERR_CONFIG, "attention inputs must be finite");  // kernels.hpp:280-283
    return TKB_OK;
}

}  // namespace

extern "C" {

TKB_API void tkb_attn_desc_init(tkb_attn_desc* d, int32_t batches, int32_t heads, int32_t seq, int32_t head_dim,
                                int32_t causal) {
    if (!d) return;
    *d = tkb_attn_desc{};
    d->batches = batches;
    d->heads = heads;
    d->seq = seq;
    d->head_dim = head_dim;
    d->causal = causal;
}

// AttentionConfig::validate (kernels.hpp:188-202), with the B200 tiling: any N >= 1
// (tails are masked), D in {64, 128}.
TKB_API int tkb_attn_validate(const tkb_attn_desc* d) {
    if (!d) return fail(TKB_ERR_BOUNDS, "null descriptor");
    if (d->head_dim != 64 && d->head_dim != 128) return fail(TKB_ERR_CONFIG, "head_dim must be 64 or 128");
    if (d->batches < 1 || d->heads < 1 || d->seq < 1) return fail(TKB_ERR_CONFIG, "positive extents required");
    if (d->causal != 0 && d->causal != 1) return fail(TKB_ERR_CONFIG, "causal must be 0 or 1");
    if (!std::isfinite(d->softmax_scale) || d->softmax_scale < 0.f)
        return fail(TKB_ERR_CONFIG, "softmax_scale must be finite and >= 0 (0: D^-1/2)");
    // the persistent schedulers index (b, h, 128-row block) tasks with 32-bit ints
    if ((int64_t)d->batches * d->heads * ((d->seq + 127) / 128) > (int64_t)INT32_MAX)
        return fail(TKB_ERR_CONFIG, "B * H * ceil(N / 128) must be < 2^31");
    if (d->kv_heads < 0 || d->heads % kv_heads_of(d) != 0)
        return fail(TKB_ERR_CONFIG, "heads must be a multiple of kv_heads (grouped-query attention)");
    for (const Strides& s : {strides_of(d), kv_strides_of(d)})
        if (s.n < d->head_dim || s.h < 0 || s.b < 0 || (s.n % 8) || (s.h % 8) || (s.b % 8))
            return fail(TKB_ERR_SHAPE, "strides must be multiples of 8 elements (16 B) with rows >= head_dim");
    return TKB_OK;
}

// Variable-length validation on top of tkb_attn_validate: packed layout (no batch strides),
// cu_seqlens present, T within the 32-bit TMA coordinate range.
static int varlen_validate(const tkb_attn_desc* d, const Varlen& vl) {
    if (!vl.cu) return fail(TKB_ERR_BOUNDS, "null cu_seqlens");
    if ((uintptr_t)vl.cu & 3) return fail(TKB_ERR_SHAPE, "cu_seqlens must be 4-byte aligned");
    if (vl.total < 0 || vl.total >= (int64_t)INT32_MAX - d->seq)
        return fail(TKB_ERR_CONFIG, "total_tokens must be in [0, 2^31 - max_seqlen)");
    if (d->stride_b != 0 || d->kv_stride_b != 0)
        return fail(TKB_ERR_SHAPE, "variable-length tensors are packed [T, H, D]: batch strides must be 0");
    for (const Strides& s : {varlen_strides(d, false), varlen_strides(d, true)})
        if (s.n < d->head_dim || (s.n % 8) || (s.h % 8))
            return fail(TKB_ERR_SHAPE, "strides must be multiples of 8 elements (16 B) with rows >= head_dim");
    return TKB_OK;
}

// With desc.check_finite (the synchronising input check) a variable-length call also reads
// cu_seqlens back and checks it: cu[0] = 0, non-decreasing, every length <= desc.seq and
// cu[B] <= total_tokens. Without it these are the caller's preconditions (no device read-back).
static int varlen_check_offsets(const tkb_attn_desc* d, const Varlen& vl, cudaStream_t st) {
    std::vector<int32_t> cu((size_t)d->batches + 1);
    cudaError_t e = cudaMemcpyAsync(cu.data(), vl.cu, cu.size() * sizeof(int32_t), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return fail(TKB_ERR_CUDA, std::string("cu_seqlens read-back: ") + cudaGetErrorString(e));
    if (cu[0] != 0) return fail(TKB_ERR_CONFIG, "cu_seqlens[0] must be 0");
    for (int b = 0; b < d->batches; ++b) {
        const int64_t n = (int64_t)cu[b + 1] - cu[b];
        if (n < 0) return fail(TKB_ERR_CONFIG, "cu_seqlens must be non-decreasing");
        if (n > d->seq) return fail(TKB_ERR_CONFIG, "a sequence is longer than desc.seq (the maximum length)");
    }
    if ((int64_t)cu[d->batches] > vl.total) return fail(TKB_ERR_BOUNDS, "cu_seqlens[B] exceeds total_tokens");
    return TKB_OK;
}

static int fwd_impl(const tkb_attn_desc* d, const Varlen* vl, const void* q, const void* k, const void* v, void* o,
             float* lse, void* workspace, size_t workspace_bytes, void* stream) {
    g_launches = 0;
    int rc = tkb_attn_validate(d);
    if (rc) return rc;
    if (vl && (rc = varlen_validate(d, *vl))) return rc;
    if (vl && (!workspace || workspace_bytes < round256(varlen_map_bytes(d, tkb::kFwdMaps))))
        return fail(TKB_ERR_BOUNDS, "varlen workspace missing or too small");
    if (vl && ((uintptr_t)workspace & 127)) return fail(TKB_ERR_SHAPE, "varlen workspace must be 128-byte aligned");
    if (!q || !k || !v || !o) return fail(TKB_ERR_BOUNDS, "null tensor pointer");
    if (((uintptr_t)q | (uintptr_t)k | (uintptr_t)v | (uintptr_t)o) & 15)
        return fail(TKB_ERR_SHAPE, "tensors must be 16-byte aligned");
    if ((rc = check_device())) return rc;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const Strides s = vl ? varlen_strides(d, false) : strides_of(d);
    const Strides skv = vl ? varlen_strides(d, true) : kv_strides_of(d);
    const int hkv = kv_heads_of(d);
    int sms = 0, *slot = nullptr;
    if ((rc = device_state(st, &sms, &slot))) return rc;
    if (d->check_finite) {
        const void* qp[1] = {q};
        const void* kvp[2] = {k, v};
        if ((vl && (rc = varlen_check_offsets(d, *vl, st))) || (rc = finite_check(d, qp, 1, s, d->heads, slot, st, vl)) ||
            (rc = finite_check(d, kvp, 2, skv, hkv, slot, st, vl)))
            return rc;
    }
    tkb::FwdParams p{};
    int launches = 1;
    if (vl) {  // per-sequence maps into the workspace (one small launch ahead of the attention)
        tkb::VarlenMapTemplates t{};
        t.nmaps = tkb::kFwdMaps;
        if ((rc = varlen_template(&t, tkb::kMapQ, q, d, s, d->heads)) ||
            (rc = varlen_template(&t, tkb::kMapK, k, d, skv, hkv)) ||
            (rc = varlen_template(&t, tkb::kMapV, v, d, skv, hkv)) ||
            (rc = varlen_template(&t, tkb::kMapO, o, d, s, d->heads)) ||
            (rc = varlen_maps(t, *vl, d->batches, workspace, st)))
            return rc;
        p.tm_q = t.tmpl[tkb::kMapQ], p.tm_k = t.tmpl[tkb::kMapK], p.tm_v = t.tmpl[tkb::kMapV], p.tm_o = t.tmpl[tkb::kMapO];
        p.vmaps = reinterpret_cast<const CUtensorMap*>(workspace);
        ++launches;
    } else if ((rc = make_bhnd_map(&p.tm_q, q, d, s)) || (rc = make_bhnd_map(&p.tm_k, k, d, skv, hkv)) ||
               (rc = make_bhnd_map(&p.tm_v, v, d, skv, hkv)) || (rc = make_bhnd_map(&p.tm_o, o, d, s))) {
        return rc;
    }
    p.cu_seqlens = vl ? vl->cu : nullptr;
    p.group = d->heads / hkv;
    p.sched = slot;
    p.lse = lse;
    p.trace = g_trace;
    p.trace_every = g_trace_every;
    p.trace_slots = g_trace_slots;
    p.n = d->seq;
    p.heads = d->heads;
    p.scale_log2 = scale_of(d) * 1.44269504088896340736f;
    p.task_tiles = g_fwd_task_tiles;
    int e = tkb::launch_attn_fwd(d->head_dim, d->causal != 0, p, d->batches, sms, st);
    if (e != 0) return fail(TKB_ERR_CUDA, std::string("attn_fwd launch: ") + cudaGetErrorString((cudaError_t)e));
    g_launches = launches;
    return TKB_OK;
}

TKB_API int tkb_attn_fwd(const tkb_attn_desc* d, const void* q, const void* k, const void* v, void* o, float* lse,
                         void* stream) {
    return fwd_impl(d, nullptr, q, k, v, o, lse, nullptr, 0, stream);
}

TKB_API size_t tkb_attn_fwd_varlen_workspace_bytes(const tkb_attn_desc* d) {
    if (!d || d->batches < 1) return 0;
    return round256(varlen_map_bytes(d, tkb::kFwdMaps));
}

TKB_API int tkb_attn_fwd_varlen(const tkb_attn_desc* d, const int32_t* cu_seqlens, int64_t total_tokens,
                                const void* q, const void* k, const void* v, void* o, float* lse, void* workspace,
                                size_t workspace_bytes, void* stream) {
    const Varlen vl{cu_seqlens, total_tokens};
    return fwd_impl(d, &vl, q, k, v, o, lse, workspace, workspace_bytes, stream);
}

// Fused rotary + forward (the rotary prologue of SURVEY §8(f) rank 2 folded into the forward
// launch): flags of the rotated blocks live in a caller-provided workspace, cleared on the
// stream before each launch (so any contents are fine and a captured graph replays correctly).
TKB_API size_t tkb_attn_fwd_rotary_workspace_bytes(const tkb_attn_desc* d) {
    if (!d || d->seq < 1 || d->batches < 1 || d->heads < 1) return 0;
    const size_t nq = (size_t)(d->seq + 127) / 128;
    const size_t hkv = (size_t)kv_heads_of(d);
    const size_t bytes = 4 * nq * (size_t)d->batches * (hkv + (size_t)d->heads);
    return (bytes + 255) & ~(size_t)255;
}

TKB_API int tkb_attn_fwd_rotary(const tkb_attn_desc* d, const void* q, const void* k, const void* v,
                                const float* sin_tab, const float* cos_tab, void* q_rot, void* k_rot, void* o,
                                float* lse, void* workspace, size_t workspace_bytes, void* stream) {
    g_launches = 0;
    int rc = tkb_attn_validate(d);
    if (rc) return rc;
    if (!q || !k || !v || !o || !sin_tab || !cos_tab || !q_rot || !k_rot || !workspace)
        return fail(TKB_ERR_BOUNDS, "null pointer");
    if (workspace_bytes < tkb_attn_fwd_rotary_workspace_bytes(d)) return fail(TKB_ERR_BOUNDS, "workspace too small");
    if (((uintptr_t)q | (uintptr_t)k | (uintptr_t)v | (uintptr_t)o | (uintptr_t)q_rot | (uintptr_t)k_rot |
         (uintptr_t)sin_tab | (uintptr_t)cos_tab | (uintptr_t)workspace) &
        15)
        return fail(TKB_ERR_SHAPE, "tensors must be 16-byte aligned");
    if (q_rot == q || k_rot == k) return fail(TKB_ERR_CONFIG, "q_rot / k_rot must not alias q / k");
    if ((rc = check_device())) return rc;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const Strides s = strides_of(d);
    const Strides skv = kv_strides_of(d);
    const int hkv = kv_heads_of(d);
    int sms = 0, *slot = nullptr;
    if ((rc = device_state(st, &sms, &slot))) return rc;
    if (d->check_finite) {
        const void* qp[1] = {q};
        const void* kvp[2] = {k, v};
        if ((rc = finite_check(d, qp, 1, s, d->heads, slot, st)) ||
            (rc = finite_check(d, kvp, 2, skv, hkv, slot, st)))
            return rc;
    }
    tkb::FwdParams p{};
    // the attention reads the rotated copies through TMA
    if ((rc = make_bhnd_map(&p.tm_q, q_rot, d, s)) || (rc = make_bhnd_map(&p.tm_k, k_rot, d, skv, hkv)) ||
        (rc = make_bhnd_map(&p.tm_v, v, d, skv, hkv)) || (rc = make_bhnd_map(&p.tm_o, o, d, s)))
        return rc;
    p.group = d->heads / hkv;
    p.sched = slot;
    p.lse = lse;
    p.trace = g_trace;
    p.trace_every = g_trace_every;
    p.trace_slots = g_trace_slots;
    p.n = d->seq;
    p.heads = d->heads;
    p.scale_log2 = scale_of(d) * 1.44269504088896340736f;
    p.sin_tab = sin_tab;
    p.cos_tab = cos_tab;
    p.q_src = q;
    p.k_src = k;
    p.q_rot = q_rot;
    p.k_rot = k_rot;
    p.q_sb = s.b, p.q_sh = s.h, p.q_sn = s.n;
    p.k_sb = skv.b, p.k_sh = skv.h, p.k_sn = skv.n;
    p.flags = reinterpret_cast<unsigned*>(workspace);
    // The flags are cleared on the stream ahead of every launch and published as 1. (A per-call
    // host epoch would be frozen into a captured graph: from its second replay on, the load
    // warp would find last replay's flags already set and read stale rotated blocks.)
    p.epoch = 1;
    cudaError_t ce = cudaMemsetAsync(workspace, 0, tkb_attn_fwd_rotary_workspace_bytes(d), st);
    if (ce != cudaSuccess) return fail(TKB_ERR_CUDA, std::string("rotary flags: ") + cudaGetErrorString(ce));
    p.task_tiles = g_fwd_task_tiles;
    const int err = tkb::launch_attn_fwd(d->head_dim, d->causal != 0, p, d->batches, sms, st, true);
    if (err != 0) return fail(TKB_ERR_CUDA, std::string("attn_fwd (rotary) launch: ") + cudaGetErrorString((cudaError_t)err));
    g_launches = 1;
    return TKB_OK;
}

TKB_API size_t tkb_attn_bwd_workspace_bytes(const tkb_attn_desc* d) {
    if (!d || d->seq < 1 || d->batches < 1 || d->heads < 1) return 0;
    const size_t bh = (size_t)d->batches * d->heads;
    const size_t npad = (size_t)((d->seq + 127) / 128) * 128;
    size_t bytes = 0;
    bytes += bh * npad * 4;  // delta = rowsum(dO * O)
    bytes += bh * npad * 4;  // lse2 (log2 domain, padded)
    const int hkv = kv_heads_of(d);
    if (hkv > 0 && d->heads % hkv == 0) {  // grouped-query split: fp32 dV / dK partials per chunk
        const size_t units = (size_t)d->batches * hkv;
        const int split = tkb::bwd_kv_split((long long)units, d->heads / hkv, (int)(npad / 128), false);
        if (split > 1) bytes += 2 * (size_t)split * units * npad * d->head_dim * 4;
    }
    return (bytes + 255) & ~(size_t)255;
}

static int bwd_impl(const tkb_attn_desc* d, const Varlen* vl, const void* q, const void* k, const void* v, const void* o,
             const void* dout, const float* lse, void* dq, void* dk, void* dv, void* workspace, size_t workspace_bytes,
             void* stream) {
    g_launches = 0;
    int rc = tkb_attn_validate(d);
    if (rc) return rc;
    if (vl && (rc = varlen_validate(d, *vl))) return rc;
    if (!q || !k || !v || !o || !dout || !lse || !dq || !dk || !dv || !workspace)
        return fail(TKB_ERR_BOUNDS, "null pointer");
    const size_t map_bytes = vl ? round256(varlen_map_bytes(d, tkb::kBwdMaps)) : 0;  // per-sequence maps first
    if (workspace_bytes < tkb_attn_bwd_workspace_bytes(d) + map_bytes)
        return fail(TKB_ERR_BOUNDS, "workspace too small");
    if (vl && ((uintptr_t)workspace & 127)) return fail(TKB_ERR_SHAPE, "varlen workspace must be 128-byte aligned");
    if (((uintptr_t)q | (uintptr_t)k | (uintptr_t)v | (uintptr_t)o | (uintptr_t)dout | (uintptr_t)dq |
         (uintptr_t)dk | (uintptr_t)dv | (uintptr_t)workspace) &
        15)
        return fail(TKB_ERR_SHAPE, "tensors must be 16-byte aligned");
    if ((rc = check_device())) return rc;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const Strides s = vl ? varlen_strides(d, false) : strides_of(d);
    const Strides skv = vl ? varlen_strides(d, true) : kv_strides_of(d);
    const int hkv = kv_heads_of(d);
    int sms = 0, *slot = nullptr;
    if ((rc = device_state(st, &sms, &slot))) return rc;
    if (d->check_finite) {
        const void* qp[3] = {q, o, dout};
        const void* kvp[2] = {k, v};
        if ((vl && (rc = varlen_check_offsets(d, *vl, st))) || (rc = finite_check(d, qp, 3, s, d->heads, slot, st, vl)) ||
            (rc = finite_check(d, kvp, 2, skv, hkv, slot, st, vl)))
            return rc;
    }
    tkb::BwdParams p{};
    int map_launches = 0;
    if (vl) {  // per-sequence maps at the start of the workspace (one small launch ahead)
        tkb::VarlenMapTemplates t{};
        t.nmaps = tkb::kBwdMaps;
        if ((rc = varlen_template(&t, tkb::kMapQ, q, d, s, d->heads)) ||
            (rc = varlen_template(&t, tkb::kMapK, k, d, skv, hkv)) ||
            (rc = varlen_template(&t, tkb::kMapV, v, d, skv, hkv)) ||
            (rc = varlen_template(&t, tkb::kMapDo, dout, d, s, d->heads)) ||
            (rc = varlen_template(&t, tkb::kMapDq, dq, d, s, d->heads)) ||
            (rc = varlen_template(&t, tkb::kMapDk, dk, d, skv, hkv)) ||
            (rc = varlen_template(&t, tkb::kMapDv, dv, d, skv, hkv)) ||
            (rc = varlen_maps(t, *vl, d->batches, workspace, st)))
            return rc;
        p.tm_q = t.tmpl[tkb::kMapQ], p.tm_k = t.tmpl[tkb::kMapK], p.tm_v = t.tmpl[tkb::kMapV];
        p.tm_do = t.tmpl[tkb::kMapDo], p.tm_dq = t.tmpl[tkb::kMapDq], p.tm_dk = t.tmpl[tkb::kMapDk];
        p.tm_dv = t.tmpl[tkb::kMapDv];
        p.vmaps = reinterpret_cast<const CUtensorMap*>(workspace);
        workspace = static_cast<char*>(workspace) + map_bytes;
        map_launches = 1;
    } else if ((rc = make_bhnd_map(&p.tm_q, q, d, s)) || (rc = make_bhnd_map(&p.tm_k, k, d, skv, hkv)) ||
               (rc = make_bhnd_map(&p.tm_v, v, d, skv, hkv)) || (rc = make_bhnd_map(&p.tm_do, dout, d, s)) ||
               (rc = make_bhnd_map(&p.tm_dq, dq, d, s)) || (rc = make_bhnd_map(&p.tm_dk, dk, d, skv, hkv)) ||
               (rc = make_bhnd_map(&p.tm_dv, dv, d, skv, hkv)) || (rc = make_bhnd_map(&p.tm_q64, q, d, s, 0, 64)) ||
               (rc = make_bhnd_map(&p.tm_do64, dout, d, s, 0, 64))) {
        return rc;
    }
    p.cu_seqlens = vl ? vl->cu : nullptr;
    p.group = d->heads / hkv;
    const int64_t bh = (int64_t)d->batches * d->heads;
    const int npad = (d->seq + 127) / 128 * 128;
    float* delta = reinterpret_cast<float*>(workspace);
    float* lse2 = delta + (size_t)bh * npad;
    p.delta = delta;
    p.lse2 = lse2;
    p.trace = g_trace;
    p.trace_every = g_trace_every;
    p.trace_slots = g_trace_slots;
    p.n = d->seq;
    p.n_pad = npad;
    p.heads = d->heads;
    p.scale = scale_of(d);
    p.scale_log2 = p.scale * 1.44269504088896340736f;
    {
        p.sched = slot;
        p.num_sms = sms;
        p.bh = (int)bh;
        // heads whose K / V (4 N D bytes each) fit in ~48 MB of L2 run together
        const long long kv_bytes = 4ll * d->seq * d->head_dim;
        long long hg = (48ll << 20) / (kv_bytes > 0 ? kv_bytes : 1);
        p.head_group = (int)(hg < 1 ? 1 : (hg > bh ? bh : hg));
    }
    p.pairs = g_bwd_pairs;
    p.kv_split = tkb::bwd_kv_split((long long)d->batches * hkv, p.group, npad / 128, vl != nullptr);
    p.dkv_part = p.kv_split > 1 ? lse2 + (size_t)bh * npad : nullptr;
    tkb::fill_bwd_divisors(p);
    p.dk = dk;
    p.dv = dv;
    p.kv_sb = skv.b;
    p.kv_sh = skv.h;
    p.kv_sn = skv.n;
    p.dq = dq;
    p.q_sb = s.b;
    p.q_sh = s.h;
    p.q_sn = s.n;
    int launches = 0;
    int e = tkb::launch_attn_bwd(d->head_dim, d->causal != 0, p, d->batches, o, dout, lse, lse2, delta, s.b, s.h,
                                 s.n, st, g_bwd_phases, &launches);
    if (e != 0) return fail(TKB_ERR_CUDA, std::string("attn_bwd launch: ") + cudaGetErrorString((cudaError_t)e));
    g_launches = launches + map_launches;
    return TKB_OK;
}

TKB_API int tkb_attn_bwd(const tkb_attn_desc* d, const void* q, const void* k, const void* v, const void* o,
                         const void* dout, const float* lse, void* dq, void* dk, void* dv, void* workspace,
                         size_t workspace_bytes, void* stream) {
    return bwd_impl(d, nullptr, q, k, v, o, dout, lse, dq, dk, dv, workspace, workspace_bytes, stream);
}

TKB_API size_t tkb_attn_bwd_varlen_workspace_bytes(const tkb_attn_desc* d) {
    const size_t b = tkb_attn_bwd_workspace_bytes(d);
    return b ? b + round256(varlen_map_bytes(d, tkb::kBwdMaps)) : 0;
}

TKB_API int tkb_attn_bwd_varlen(const tkb_attn_desc* d, const int32_t* cu_seqlens, int64_t total_tokens,
                                const void* q, const void* k, const void* v, const void* o, const void* dout,
                                const float* lse, void* dq, void* dk, void* dv, void* workspace, size_t workspace_bytes,
                                void* stream) {
    const Varlen vl{cu_seqlens, total_tokens};
    return bwd_impl(d, &vl, q, k, v, o, dout, lse, dq, dk, dv, workspace, workspace_bytes, stream);
}

// RotaryConfig::validate (kernels.hpp:367-376) relaxed to the B200 layout: even head_dim,
// a multiple of 16 (8-pair vectors), any seq >= 1.
int rotary_validate(const tkb_attn_desc* d) {
    if (!d) return fail(TKB_ERR_BOUNDS, "null descriptor");
    if (d->batches < 1 || d->heads < 1 || d->seq < 1) return fail(TKB_ERR_CONFIG, "positive extents required");
    if (d->head_dim < 16 || d->head_dim % 16) return fail(TKB_ERR_CONFIG, "rotary head_dim must be a multiple of 16");
    if (d->kv_heads < 0 || d->heads % kv_heads_of(d)) return fail(TKB_ERR_CONFIG, "heads % kv_heads != 0");
    for (const Strides& s : {strides_of(d), kv_strides_of(d)})
        if (s.n < d->head_dim || (s.n % 8) || (s.h % 8) || (s.b % 8))
            return fail(TKB_ERR_SHAPE, "strides must be multiples of 8 elements with rows >= head_dim");
    return TKB_OK;
}

tkb::rope::Tensor rope_tensor(const tkb_attn_desc* d, const void* x, void* o, const Strides& s, int heads) {
    tkb::rope::Tensor t;
    t.x = x;
    t.o = o;
    t.xb = t.ob = s.b;
    t.xh = t.oh = s.h;
    t.xn = t.on = s.n;
    t.heads = heads;
    t.items = (int64_t)d->batches * heads * d->seq * (d->head_dim / 16);
    return t;
}

// Rotary embedding (rotary_kernel, kernels.hpp:413-503): out = rotate(x) by fp32 [seq, head_dim/2]
// sin / cos tables. x, out: [B, H, N, D] bf16 with desc's strides (out may alias x).
TKB_API int tkb_rotary(const tkb_attn_desc* d, const void* x, const float* sin_tab, const float* cos_tab, void* out,
                       void* stream) {
    g_launches = 0;
    int rc = rotary_validate(d);
    if (rc) return rc;
    if (!x || !sin_tab || !cos_tab || !out) return fail(TKB_ERR_BOUNDS, "null pointer");
    if (((uintptr_t)x | (uintptr_t)out | (uintptr_t)sin_tab | (uintptr_t)cos_tab) & 15)
        return fail(TKB_ERR_SHAPE, "tensors must be 16-byte aligned");
    if ((rc = check_device())) return rc;
    int sms = 0;
    if ((rc = device_state(reinterpret_cast<cudaStream_t>(stream), &sms, nullptr))) return rc;
    tkb::rope::Params p{};
    p.t[0] = rope_tensor(d, x, out, strides_of(d), d->heads);
    p.sin_tab = sin_tab;
    p.cos_tab = cos_tab;
    p.n = d->seq;
    p.hd = d->head_dim;
    const int e = tkb::launch_rotary(p, sms, reinterpret_cast<cudaStream_t>(stream));
    if (e) return fail(TKB_ERR_CUDA, std::string("rotary launch: ") + cudaGetErrorString((cudaError_t)e));
    g_launches = 1;
    return TKB_OK;
}

// The attention prologue: Q ([B, H, N, D], desc strides) and K ([B, Hkv, N, D], kv strides)
// rotated in one launch into q_out / k_out (which may alias q / k).
TKB_API int tkb_rotary_qk(const tkb_attn_desc* d, const void* q, const void* k, const float* sin_tab,
                          const float* cos_tab, void* q_out, void* k_out, void* stream) {
    g_launches = 0;
    int rc = rotary_validate(d);
    if (rc) return rc;
    if (!q || !k || !sin_tab || !cos_tab || !q_out || !k_out) return fail(TKB_ERR_BOUNDS, "null pointer");
    if (((uintptr_t)q | (uintptr_t)k | (uintptr_t)q_out | (uintptr_t)k_out | (uintptr_t)sin_tab |
         (uintptr_t)cos_tab) &
        15)
        return fail(TKB_ERR_SHAPE, "tensors must be 16-byte aligned");
    if ((rc = check_device())) return rc;
    int sms = 0;
    if ((rc = device_state(reinterpret_cast<cudaStream_t>(stream), &sms, nullptr))) return rc;
    tkb::rope::Params p{};
    p.t[0] = rope_tensor(d, q, q_out, strides_of(d), d->heads);
    p.t[1] = rope_tensor(d, k, k_out, kv_strides_of(d), kv_heads_of(d));
    p.sin_tab = sin_tab;
    p.cos_tab = cos_tab;
    p.n = d->seq;
    p.hd = d->head_dim;
    const int e = tkb::launch_rotary(p, sms, reinterpret_cast<cudaStream_t>(stream));
    if (e) return fail(TKB_ERR_CUDA, std::string("rotary launch: ") + cudaGetErrorString((cudaError_t)e));
    g_launches = 1;
    return TKB_OK;
}

// GemmConfig::validate (kernels.hpp:33-41) relaxed to the B200 layout: any m, n, k >= 1
// (ragged edges are zero-filled / clipped by TMA), row strides multiples of 8 elements.
TKB_API int tkb_gemm_validate(const tkb_gemm_desc* d) {
    if (!d) return fail(TKB_ERR_BOUNDS, "null descriptor");
    if (d->m < 1 || d->n < 1 || d->k < 1) return fail(TKB_ERR_CONFIG, "GEMM extents must be positive");
    if (d->super_m < 0) return fail(TKB_ERR_CONFIG, "super_m must be >= 1 (0: default 12)");
    const int64_t lda = d->lda ? d->lda : d->k, ldb = d->ldb ? d->ldb : d->n, ldc = d->ldc ? d->ldc : d->n;
    if (lda < d->k || ldb < d->n || ldc < d->n || (lda % 8) || (ldb % 8) || (ldc % 8))
        return fail(TKB_ERR_SHAPE, "row strides must be multiples of 8 elements covering the rows");
    return TKB_OK;
}

TKB_API int tkb_gemm(const tkb_gemm_desc* d, const void* a, const void* b, void* c, void* stream) {
    g_launches = 0;
    int rc = tkb_gemm_validate(d);
    if (rc) return rc;
    if (!a || !b || !c) return fail(TKB_ERR_BOUNDS, "null tensor pointer");
    if (((uintptr_t)a | (uintptr_t)b | (uintptr_t)c) & 15) return fail(TKB_ERR_SHAPE, "tensors must be 16-byte aligned");
    if ((rc = check_device())) return rc;
    int sms = 0;
    if ((rc = device_state(reinterpret_cast<cudaStream_t>(stream), &sms, nullptr))) return rc;
    const uint64_t lda = d->lda ? d->lda : d->k, ldb = d->ldb ? d->ldb : d->n, ldc = d->ldc ? d->ldc : d->n;
    tkb::GemmParams p{};
    std::string err;
    {
        uint64_t dims[2] = {(uint64_t)d->k, (uint64_t)d->m}, str[2] = {1, lda};
        uint32_t box[2] = {64, 128};
        if (!tkb::host::make_tmap(&p.tm_a, a, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, 2, dims, str, box,
                                  CU_TENSOR_MAP_SWIZZLE_128B, &err))
            return fail(TKB_ERR_SHAPE, "tensor map A: " + err);
    }
    {
        uint64_t dims[2] = {(uint64_t)d->n, (uint64_t)d->k}, str[2] = {1, ldb};
        uint32_t box[2] = {64, 64};
        if (!tkb::host::make_tmap(&p.tm_b, b, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, 2, dims, str, box,
                                  CU_TENSOR_MAP_SWIZZLE_128B, &err))
            return fail(TKB_ERR_SHAPE, "tensor map B: " + err);
    }
    {
        uint64_t dims[2] = {(uint64_t)d->n, (uint64_t)d->m}, str[2] = {1, ldc};
        uint32_t box[2] = {64, 128};
        if (!tkb::host::make_tmap(&p.tm_c, c, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, 2, dims, str, box,
                                  CU_TENSOR_MAP_SWIZZLE_128B, &err))
            return fail(TKB_ERR_SHAPE, "tensor map C: " + err);
    }
    p.m = d->m;
    p.n = d->n;
    p.k = d->k;
    p.super_m = d->super_m > 0 ? d->super_m : 12;
    const int e = tkb::launch_gemm(p, sms, reinterpret_cast<cudaStream_t>(stream));
    if (e) return fail(TKB_ERR_CUDA, std::string("gemm launch: ") + cudaGetErrorString((cudaError_t)e));
    g_launches = 1;
    return TKB_OK;
}

TKB_API int tkb_shard_range(int64_t units, int32_t rank, int32_t world, int64_t* begin, int64_t* end) {
    if (!begin || !end) return fail(TKB_ERR_BOUNDS, "null output");
    if (world < 1 || rank < 0 || rank >= world || units < 0) return fail(TKB_ERR_CONFIG, "bad rank/world/units");
    const int64_t base = units / world, rem = units % world;
    *begin = rank * base + (rank < rem ? rank : rem);
    *end = *begin + base + (rank < rem ? 1 : 0);
    return TKB_OK;
}

TKB_API int tkb_debug_set_trace(void* device_buf, int every, int slots) {
    g_trace = reinterpret_cast<long long*>(device_buf);
    g_trace_every = every > 0 ? every : 1;
    g_trace_slots = device_buf ? slots : 0;
    return TKB_OK;
}

TKB_API int tkb_debug_set_bwd_phases(int mask) {
    g_bwd_phases = mask & 7;
    return TKB_OK;
}

TKB_API int tkb_set_bwd_pairs(int on) {
    g_bwd_pairs = on ? 1 : 0;
    return TKB_OK;
}

TKB_API int tkb_debug_set_fwd_task_tiles(int tiles) {
    if (tiles < 0 || tiles > 2) return fail(TKB_ERR_CONFIG, "forward task tiles must be 0 (auto), 1 or 2");
    g_fwd_task_tiles = tiles;
    return TKB_OK;
}

TKB_API int tkb_device_init(int device) {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess) return fail(TKB_ERR_CUDA, std::string("cudaGetDeviceCount: ") + cudaGetErrorString(e));
    if (device < 0 || device >= n) return fail(TKB_ERR_CONFIG, "no such device");
    return device_init(device);
}

TKB_API int tkb_debug_map_cache_stats(unsigned long long* hits, unsigned long long* misses) {
    if (hits) *hits = g_map_hits;
    if (misses) *misses = g_map_misses;
    return TKB_OK;
}

TKB_API int tkb_last_launch_count(void) { return g_launches; }
TKB_API const char* tkb_last_error(void) { return g_err.c_str(); }
TKB_API int tkb_abi_version(void) { return TKB_ABI_VERSION; }

}  // extern "C"
