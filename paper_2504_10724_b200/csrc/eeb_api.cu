// eeb_api.cu — context, model registry, greedy layer loader and the batched
// early-exit decode step behind the C ABI in include/eeb/eeb.h.
//
// The step is the batched form of Simulator::serve_one's token loop
// (/root/reference/proj/include/eeserve/engine.hpp:344-386):
// one call advances every row one token.  The launch sequence for a given
// (model, depth, policy, batch) is fixed — row counts after compaction live
// in device memory — so it is captured once into a CUDA graph and replayed.
#include <cuda.h>
#include <dlfcn.h>
#include <nccl.h>
#include <cublasLt.h>

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <set>
#include <memory>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/eeb/eeb.h"
#include "kernels.h"
#include "synth.cuh"

namespace eeb {

namespace {

thread_local std::string g_last_error;

// Device block cache for model weights.  The greedy loader evicts and reloads
// layers as the served model and depth change; cudaMalloc / cudaFree of those
// GBs cost ~1 s of host time per C3 serving run (and every cudaFree
// synchronises the device).  Evicted weight buffers are kept here and handed
// to the next allocation of the same size; an allocation that fails anywhere
// in the library first returns every pool's blocks to the driver.
struct BlockPool;
std::mutex g_pools_mu;
std::vector<BlockPool*> g_pools;
struct BlockPool {
    std::mutex mu;
    std::multimap<size_t, void*> blocks;
    BlockPool() {
        std::lock_guard<std::mutex> g(g_pools_mu);
        g_pools.push_back(this);
    }
    ~BlockPool() {
        {
            std::lock_guard<std::mutex> g(g_pools_mu);
            g_pools.erase(std::find(g_pools.begin(), g_pools.end(), this));
        }
        trim();
    }
    BlockPool(const BlockPool&) = delete;
    BlockPool& operator=(const BlockPool&) = delete;
    void trim() {
        std::lock_guard<std::mutex> g(mu);
        for (auto& kv : blocks) cudaFree(kv.second);
        blocks.clear();
    }
    void* take(size_t n) {
        std::lock_guard<std::mutex> g(mu);
        const auto it = blocks.find(n);
        if (it == blocks.end()) return nullptr;
        void* q = it->second;
        blocks.erase(it);
        return q;
    }
    void put(void* q, size_t n) {
        std::lock_guard<std::mutex> g(mu);
        blocks.emplace(n, q);
    }
};
void dev_malloc(void** q, size_t n) {
    cudaError_t e = cudaMalloc(q, n);
    if (e == cudaErrorMemoryAllocation) {
        cudaGetLastError();
        {
            std::lock_guard<std::mutex> g(g_pools_mu);
            for (BlockPool* bp : g_pools) bp->trim();
        }
        e = cudaMalloc(q, n);
    }
    EEB_CUDA(e);
}

struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    BlockPool* pool = nullptr;  // weights: blocks recycled through the context's pool
    DevBuf() = default;
    explicit DevBuf(BlockPool* bp) : pool(bp) {}
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { release(); }
    void release() {
        if (p) {
            if (pool) pool->put(p, bytes);
            else cudaFree(p);
        }
        p = nullptr;
        bytes = 0;
    }
    // Returns true when the buffer moved (captured graphs holding it are stale).
    bool ensure(size_t n) {
        if (n <= bytes) return false;
        release();
        p = pool ? pool->take(n) : nullptr;
        if (!p) dev_malloc(&p, n);
        bytes = n;
        // debugging aid: fill fresh allocations with NaN-ish bytes so reads of
        // never-written memory show up deterministically
        static const bool poison = std::getenv("EEB_DEBUG_POISON") != nullptr;
        if (poison) EEB_CUDA(cudaMemset(p, 0xFF, n));
        return true;
    }
    template <typename T> T* as() const { return static_cast<T*>(p); }
};

struct LayerWeights {
    DevBuf attn_norm, mlp_norm, wqkv, wo, wup, wdown;
    DevBuf* parts[6] = {&attn_norm, &mlp_norm, &wqkv, &wo, &wup, &wdown};
    explicit LayerWeights(BlockPool* bp) {
        for (DevBuf* b : parts) b->pool = bp;
    }
};

// Pinned host memory (the host tier the greedy loader copies from).
struct HostBuf {
    void* p = nullptr;
    size_t bytes = 0;
    HostBuf() = default;
    HostBuf(const HostBuf&) = delete;
    HostBuf& operator=(const HostBuf&) = delete;
    ~HostBuf() {
        if (p) cudaFreeHost(p);
    }
    void alloc(size_t n) {
        EEB_CUDA(cudaMallocHost(&p, n));
        bytes = n;
    }
};

// One layer (or the base weights) as a packed pinned blob: part k at off[k].
struct HostBlob {
    HostBuf buf;
    std::vector<size_t> off, sz;
};

// A model's weights in host memory ↔ the "model in CPU memory" that HELIOS's
// greedy loader pulls layers from (engine.hpp:197-216, memory_model.hpp:76-105).
struct HostTier {
    std::unique_ptr<HostBlob> base;                  // embedding, exit heads, head norms
    std::vector<std::unique_ptr<HostBlob>> layers;   // index l-1
};

// An asynchronous load in flight on the context's load stream.
struct PendingLoad {
    cudaEvent_t t0 = nullptr, t1 = nullptr;          // timing (load stream)
    std::vector<std::pair<int, cudaEvent_t>> ready;  // (layer, event); layer 0 = base weights
    int64_t bytes = 0;
};

struct Model {
    eeb_model_desc desc{};
    std::vector<int> exits;
    std::vector<float> coverage;
    std::vector<float> alphas;
    int head_dim = 0, dq = 0, dkv = 0, up_rows = 0;
    size_t wbytes = 0;  // weight element size
    // Tensor parallelism (Megatron layout): column-parallel QKV / up, row-parallel
    // O / down (partials summed across ranks), vocab-parallel exit heads.  A rank
    // context holds one shard (tp_rank >= 0, NCCL between ranks); tp_rank = -1
    // holds all tp shards in one context and sums them locally (single-GPU
    // emulation of the group: same kernels, same shard weights).
    int tp = 1, rank = 0, shards = 1;
    int hq_l = 0, hkv_l = 0, dq_l = 0, dkv_l = 0, f_l = 0, up_l = 0, v_l = 0;  // per-shard dims
    int shard_rank(int s) const { return rank >= 0 ? rank : s; }
    size_t kv_shard_elems = 0;  // one (layer, shard) block of the KV cache
    BlockPool* pool = nullptr;  // the context's weight block cache (set at registration)
    // base weights
    DevBuf emb;
    std::vector<std::unique_ptr<DevBuf>> head, head_norm;
    std::vector<std::unique_ptr<LayerWeights>> layers;  // index l-1
    int loaded = 0;
    // KV pool
    DevBuf k_cache, v_cache, kv_depth, rope_cos, rope_sin;
    size_t kv_layer_elems = 0;
    // KV pages.  Unpaged (default): one page per slot of
    // max_seq_len positions, identity table.  Paged (eeb_kv_configure_pages):
    // n_pages pages of page_size positions on a free list; a slot's table row
    // grows as its positions do and is released with the slot.
    int kv_page = 0, kv_pages = 0, pages_per_seq = 1;
    bool paged = false;
    DevBuf page_table;                 // int32 [max_slots][pages_per_seq]
    std::vector<int32_t> h_table;      // host mirror
    std::vector<int32_t> slot_npages;  // pages held per slot
    std::vector<int32_t> free_pages;   // LIFO free list
    bool table_dirty = false;
    std::vector<std::array<uint8_t, 128>> k_maps, v_maps;  // bf16: per-layer TMA maps of the KV cache (32-row boxes)
    std::vector<std::array<uint8_t, 128>> k_maps8, v_maps8;  // the same with 8-row boxes (a pass's last chunk)
    // host tier + asynchronous loader state
    HostTier host;
    std::unique_ptr<PendingLoad> pending;
    double last_load_s = 0.0;
    int64_t last_load_bytes = 0;
    // peer-memory tensor parallelism (eeb_tp_px_alloc / eeb_tp_px_attach):
    // this rank's exchange buffer and every rank's, as mapped here
    DevBuf px;
    PxPeers pxp;
    std::vector<void*> px_opened;  // CUDA IPC mappings of peer buffers
    bool px_on() const { return pxp.nranks > 1; }
    Model() = default;
    Model(const Model&) = delete;
    Model& operator=(const Model&) = delete;
    ~Model() {
        for (void* q : px_opened) cudaIpcCloseMemHandle(q);
    }
};

struct GraphKey {
    int model, depth, policy, batch, tier;
    uint32_t th_bits;
    bool operator<(const GraphKey& o) const {
        return std::tie(model, depth, policy, batch, tier, th_bits) <
               std::tie(o.model, o.depth, o.policy, o.batch, o.tier, o.th_bits);
    }
};

enum Cat { kCatGemm = 0, kCatAttn, kCatHead, kCatNorm, kCatOther, kNumCat };

const char* kCatNames[kNumCat] = {"layer_gemm", "attention", "exit_head", "norm", "other"};

}  // namespace

}  // namespace eeb

struct eeb_ctx {
    eeb::BlockPool wpool;  // first member: outlives every model's weight buffers
    int device = 0;
    int num_sms = 148;
    cudaStream_t stream = nullptr;
    cudaStream_t load_stream = nullptr;  // greedy loader: pinned H2D copies, overlapped with decode
    cudaStream_t main_stream = nullptr;  // `stream` while a conditional body is being captured
    std::vector<cudaStream_t> cond_streams;  // capture streams of nested conditional bodies (step graphs)
    bool capturing = false;               // enqueue_step runs under stream capture
    bool in_prefill = false;              // enqueue_prefill: the layer GEMMs may take cuBLASLt
    // Prefill GEMMs (plain [rows x K] x [K x N] products of every prompt row,
    // no early exit to skip): cuBLASLt, one plan per shape.
    cublasLtHandle_t lt = nullptr;
    eeb::DevBuf lt_ws;
    struct LtPlan {
        cublasLtMatmulDesc_t op = nullptr;
        cublasLtMatrixLayout_t a = nullptr, b = nullptr, d = nullptr;
        cublasLtMatmulAlgo_t algo{};
        bool ok = false;
    };
    std::map<std::tuple<int, int, int, int>, LtPlan> lt_plans;  // (N, K, rows, relu-bf16 epilogue)
    size_t cond_open = 0;                 // conditional bodies open in the capture
    std::vector<std::unique_ptr<eeb::Model>> models;
    int graphs_enabled = 1;
    int gemm_tier = 0;
    int retain_logits = 0;
    // the next tensor-core GEMM's weights, prefetched into L2 by the current one
    const void* pf_ptr = nullptr;
    size_t pf_bytes = 0;
    // plane output redirected into a TP exchange buffer (PxPlanesScope)
    float* gemm_out = nullptr;
    int64_t gemm_out_elems = 0;
    // step workspace (grow-only)
    int cap_rows = 0;
    eeb::DevBuf xA, xB, hn, hnB, hhead, attn, mlp_h, ws;
    eeb::DevBuf rows;  // ints: nA, nB, rowA, slotA, posA, rowB, slotB, posB, src, in_tok, in_slot, in_pos
    eeb::DevBuf head_tok, head_conf, head_logp, head_tri;
    eeb::DevBuf decide_ticket;  // int, zero between decide launches
    eeb::DevBuf kv_part, kv_ticket;  // decode KV-split partials and per-(row, kv head) tickets
    eeb::DevBuf tp_partial;         // row-parallel partial sums all-reduced across TP ranks
    eeb::DevBuf pf_meta;            // prefill (tok, slot, pos) of every prompt token, then the query blocks
    eeb::DevBuf pf_items;           // the current chunk's query blocks (int4) + their count
    int pf_cur_items = 0;           // query blocks of the chunk being enqueued (graph key)
    void* pf_pin = nullptr;
    size_t pf_pin_bytes = 0;
    eeb::DevBuf o_all;  // the step's outputs, one block (OutLayout): one D2H copy per host-API step
    std::vector<std::unique_ptr<eeb::DevBuf>> logits_keep;
    int64_t ws_elems = 0;
    // pinned staging for the host-pointer API
    void* pin = nullptr;
    size_t pin_bytes = 0;
    std::map<eeb::GraphKey, cudaGraphExec_t> graphs;
    std::set<eeb::GraphKey> pf_seen;  // prefill chunk layouts run once eagerly (captured on a repeat)
    // profiling
    int profiling = 0;
    std::vector<cudaEvent_t> ev_pool;
    std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> ev_used;
    double cat_ms[eeb::kNumCat] = {0};
    int64_t cat_launches[eeb::kNumCat] = {0};
    int64_t step_launches = 0;
    int64_t steps_profiled = 0;
    ncclComm_t nccl = nullptr;
    eeb::DevBuf nccl_buf;
    // in-graph launch timeline (eeb_debug_stamps)
    int stamp_cap = 0;  // launches per step recorded (0 = off)
    eeb::DevBuf stamp_buf;
    std::map<eeb::GraphKey, std::pair<std::vector<const void*>, std::vector<int>>> stamp_kernels;  // per graph: slot -> kernel, category
    std::pair<std::vector<const void*>, std::vector<int>> stamp_last;                              // ... of the last step launched
};

namespace eeb {

namespace {


// NCCL is resolved at run time (dlopen) rather than linked: the process may
// already hold torch's bundled libnccl.so.2, and two NCCL builds under one
// soname would clash.  An already-loaded NCCL is preferred.
struct NcclApi {
    decltype(&ncclGetUniqueId) get_unique_id = nullptr;
    decltype(&ncclCommInitRank) comm_init_rank = nullptr;
    decltype(&ncclAllReduce) all_reduce = nullptr;
    decltype(&ncclAllGather) all_gather = nullptr;
    decltype(&ncclGroupStart) group_start = nullptr;
    decltype(&ncclGroupEnd) group_end = nullptr;
    decltype(&ncclCommDestroy) comm_destroy = nullptr;
    decltype(&ncclGetErrorString) error_string = nullptr;
};

const NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) {
            const char* env = std::getenv("EEB_NCCL_LIB");
            h = dlopen(env && *env ? env : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        }
        if (!h) return;
        api.get_unique_id = (decltype(api.get_unique_id))dlsym(h, "ncclGetUniqueId");
        api.comm_init_rank = (decltype(api.comm_init_rank))dlsym(h, "ncclCommInitRank");
        api.all_reduce = (decltype(api.all_reduce))dlsym(h, "ncclAllReduce");
        api.all_gather = (decltype(api.all_gather))dlsym(h, "ncclAllGather");
        api.group_start = (decltype(api.group_start))dlsym(h, "ncclGroupStart");
        api.group_end = (decltype(api.group_end))dlsym(h, "ncclGroupEnd");
        api.comm_destroy = (decltype(api.comm_destroy))dlsym(h, "ncclCommDestroy");
        api.error_string = (decltype(api.error_string))dlsym(h, "ncclGetErrorString");
    });
    if (!api.get_unique_id || !api.comm_init_rank || !api.all_reduce)
        throw Error(EEB_E_CUDA, "NCCL (libnccl.so.2) could not be loaded");
    return api;
}

int status_of(const Error& e) { return e.code; }

void set_error(const std::string& m) { g_last_error = m; }

template <typename F>
eeb_status guarded(F&& f) {
    try {
        f();
        return EEB_OK;
    } catch (const Error& e) {
        set_error(e.what());
        return static_cast<eeb_status>(status_of(e));
    } catch (const std::bad_alloc&) {
        set_error("host allocation failed");
        return EEB_E_CAPACITY;
    } catch (const std::exception& e) {
        set_error(e.what());
        return EEB_E_CUDA;
    }
}

Model& model_of(eeb_ctx* c, int m) {
    if (!c) throw Error(EEB_E_DOMAIN, "null context");
    if (m < 0 || m >= (int)c->models.size() || !c->models[m])
        throw Error(EEB_E_DOMAIN, "unknown model handle " + std::to_string(m));
    return *c->models[m];
}

std::vector<float> default_coverage(int n) {
    // Cumulative exit law of the reference's OPT-1.3B calibration: 73.0 / 4.7 /
    // 22.3 % (fixtures/FIXTURES.md:47-55); intermediate heads spread the 4.7 %.
    std::vector<float> c(n);
    for (int i = 0; i < n; ++i) {
        if (i == n - 1) c[i] = 1.0f;
        else if (n <= 2 || i == 0) c[i] = 0.73f;
        else c[i] = 0.73f + 0.047f * (float)i / (float)(n - 2);
    }
    return c;
}

void validate_desc(const eeb_model_desc& d) {
    auto bad = [](const std::string& m) { throw Error(EEB_E_VALIDATION, "model: " + m); };
    if (d.num_layers <= 0 || d.num_layers > 255) bad("num_layers must be in [1, 255]");
    if (d.d_model <= 0 || d.n_heads <= 0 || d.n_kv_heads <= 0 || d.d_ffn <= 0 || d.vocab <= 1)
        bad("dimensions must be positive");
    if (d.d_model % d.n_heads != 0) bad("d_model must be a multiple of n_heads");
    if (d.n_heads % d.n_kv_heads != 0) bad("n_heads must be a multiple of n_kv_heads");
    if (d.d_model % 256 != 0 || d.d_ffn % 256 != 0) bad("d_model and d_ffn must be multiples of 256");
    if (d.n_exits <= 0 || d.n_exits > 64 || !d.exit_layers) bad("exit_layers must be non-empty (<= 64)");
    for (int i = 0; i < d.n_exits; ++i) {
        if (d.exit_layers[i] <= 0) bad("exit layers must be positive");
        if (i > 0 && d.exit_layers[i] <= d.exit_layers[i - 1]) bad("exit_layers must be strictly increasing");
    }
    if (d.exit_layers[d.n_exits - 1] != d.num_layers) bad("last exit layer must equal num_layers");
    if (d.dtype != EEB_F32 && d.dtype != EEB_BF16) bad("dtype must be f32 or bf16");
    if (d.mlp_kind != EEB_MLP_RELU && d.mlp_kind != EEB_MLP_SWIGLU) bad("unknown mlp kind");
    if (d.max_slots <= 0 || d.max_seq_len <= 0) bad("max_slots and max_seq_len must be positive");
    if (!(d.design_th >= 0.f && d.design_th <= 1.f)) bad("design_th must be in [0,1]");
    if (d.tp_size < 0 || d.tp_size > 64) bad("tp_size must be in [0, 64]");
    if (d.tp_size > 1) {
        const int t = d.tp_size;
        if (d.tp_rank < -1 || d.tp_rank >= t) bad("tp_rank must be -1 (all shards local) or in [0, tp_size)");
        if (d.n_heads % t || d.n_kv_heads % t || d.d_ffn % t || d.vocab % t)
            bad("n_heads, n_kv_heads, d_ffn and vocab must be multiples of tp_size");
        if ((d.d_ffn / t) % 256 != 0) bad("d_ffn / tp_size must be a multiple of 256");
        if (d.dtype != EEB_BF16) bad("tensor parallelism needs bf16 weights");
    }
}

// ---------------------------------------------------------------------------
// Loader ↔ do_load / apply_load: materialise layers [loaded+1, to] (and the
// base weights on the first load); free layers deeper than `to` on shrink.
// ---------------------------------------------------------------------------
// Base weights (embedding, exit heads + their norms) materialised on device.
void synth_base(Model& m, cudaStream_t s) {
    const eeb_model_desc& d = m.desc;
    const int D = d.d_model;
    m.emb.ensure((size_t)d.vocab * D * m.wbytes);
    synth_embedding(d.dtype, m.emb.p, d.seed, d.vocab, D, s);
    m.head.clear();
    m.head_norm.clear();
    for (int e = 0; e < d.n_exits; ++e) {
        auto h = std::make_unique<DevBuf>(m.pool);
        h->ensure((size_t)m.shards * m.v_l * D * m.wbytes);  // vocab shards, shard-major
        for (int sh = 0; sh < m.shards; ++sh)
            synth_head(d.dtype, static_cast<char*>(h->p) + (size_t)sh * m.v_l * D * m.wbytes, d.seed, e, m.alphas[e],
                       d.vocab, D, s, m.shard_rank(sh) * m.v_l, m.v_l);
        auto g = std::make_unique<DevBuf>(m.pool);
        g->ensure((size_t)D * sizeof(float));
        synth_norm(g->p, d.seed, synth::base_tid(synth::kHeadNorm, e), D, s);
        m.head.push_back(std::move(h));
        m.head_norm.push_back(std::move(g));
    }
}

// Device buffers of layer l, sized but not filled.
std::unique_ptr<LayerWeights> alloc_layer(const Model& m) {
    const int D = m.desc.d_model, F = m.desc.d_ffn;
    auto L = std::make_unique<LayerWeights>(m.pool);
    L->attn_norm.ensure((size_t)D * 4);
    L->mlp_norm.ensure((size_t)D * 4);
    const size_t S = (size_t)m.shards;
    L->wqkv.ensure(S * (m.dq_l + 2 * m.dkv_l) * D * m.wbytes);
    L->wo.ensure(S * D * m.dq_l * m.wbytes);
    L->wup.ensure(S * m.up_l * D * m.wbytes);
    L->wdown.ensure(S * D * m.f_l * m.wbytes);
    (void)F;
    return L;
}

// Layer l (1-based) materialised on device from the model seed.
std::unique_ptr<LayerWeights> synth_layer(const Model& m, int l, cudaStream_t s) {
    const eeb_model_desc& d = m.desc;
    const uint64_t seed = d.seed;
    const int D = d.d_model, F = d.d_ffn;
    const float rsig = synth::residual_sigma(D, F);
    auto L = alloc_layer(m);
    synth_norm(L->attn_norm.p, seed, synth::layer_tid(l, synth::kAttnNorm), D, s);
    synth_norm(L->mlp_norm.p, seed, synth::layer_tid(l, synth::kMlpNorm), D, s);
    // Shard sh of rank g: its q heads, k heads, v heads (rows of the full
    // [dq + 2 dkv][D] QKV), its columns of O and down, its rows of up — every
    // element the same (seed, tensor, index) value as in the unsharded model.
    const size_t wb = m.wbytes;
    const int qkv_l = m.dq_l + 2 * m.dkv_l;
    for (int sh = 0; sh < m.shards; ++sh) {
        const int g = m.shard_rank(sh);
        char* q = static_cast<char*>(L->wqkv.p) + (size_t)sh * qkv_l * D * wb;
        const int tq = synth::layer_tid(l, synth::kWqkv);
        synth_linear_slice(d.dtype, q, seed, tq, m.dq_l, D, g * m.dq_l, 0, D, synth::kSigma, false, D, s);
        synth_linear_slice(d.dtype, q + (size_t)m.dq_l * D * wb, seed, tq, m.dkv_l, D, m.dq + g * m.dkv_l, 0, D,
                           synth::kSigma, false, D, s);
        synth_linear_slice(d.dtype, q + (size_t)(m.dq_l + m.dkv_l) * D * wb, seed, tq, m.dkv_l, D,
                           m.dq + m.dkv + g * m.dkv_l, 0, D, synth::kSigma, false, D, s);
        synth_linear_slice(d.dtype, static_cast<char*>(L->wo.p) + (size_t)sh * D * m.dq_l * wb, seed,
                           synth::layer_tid(l, synth::kWo), D, m.dq_l, 0, g * m.dq_l, m.dq, rsig, true, D, s);
        synth_linear_slice(d.dtype, static_cast<char*>(L->wup.p) + (size_t)sh * m.up_l * D * wb, seed,
                           synth::layer_tid(l, synth::kWup), m.up_l, D, g * m.up_l, 0, D, synth::kSigma, false, D, s);
        synth_linear_slice(d.dtype, static_cast<char*>(L->wdown.p) + (size_t)sh * D * m.f_l * wb, seed,
                           synth::layer_tid(l, synth::kWdown), D, m.f_l, 0, g * m.f_l, F, rsig, true, D, s);
    }
    return L;
}

// Host side of every pending asynchronous load has to be settled before the
// synchronous loader frees or replaces buffers the copies target.
void settle_pending(Model& m) {
    if (!m.pending) return;
    EEB_CUDA(cudaEventSynchronize(m.pending->t1));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, m.pending->t0, m.pending->t1);
    m.last_load_s = ms / 1000.0;
    m.last_load_bytes = m.pending->bytes;
    cudaEventDestroy(m.pending->t0);
    cudaEventDestroy(m.pending->t1);
    for (auto& [l, ev] : m.pending->ready) cudaEventDestroy(ev);
    m.pending.reset();
}

std::unique_ptr<LayerWeights> layer_from_host(const Model& m, int l, cudaStream_t s);
void base_from_host(Model& m, cudaStream_t s);

void load_to(eeb_ctx* c, Model& m, int to) {
    const eeb_model_desc& d = m.desc;
    if (to < 0 || to > d.num_layers)
        throw Error(EEB_E_DOMAIN, "load: depth " + std::to_string(to) + " outside [0, " +
                                      std::to_string(d.num_layers) + "]");
    settle_pending(m);
    cudaStream_t s = c->stream;
    // evicted weight blocks go back to the pool (reusable at once): nothing
    // queued on the decode stream may still read them
    EEB_CUDA(cudaStreamSynchronize(s));
    if (to == 0) {
        m.layers.clear();
        m.head.clear();
        m.head_norm.clear();
        m.emb.release();
        m.loaded = 0;
        return;
    }
    // The host tier (caller-supplied weights, or a staged copy of the synthetic
    // ones) is the source when it holds the tensor; otherwise synthesise.
    if (m.loaded == 0) {
        if (m.host.base) base_from_host(m, s);
        else synth_base(m, s);
    }
    while ((int)m.layers.size() < to) {
        const int l = (int)m.layers.size() + 1;
        m.layers.push_back(l <= (int)m.host.layers.size() ? layer_from_host(m, l, s) : synth_layer(m, l, s));
    }
    while ((int)m.layers.size() > to) m.layers.pop_back();
    m.loaded = to;
    EEB_CUDA(cudaStreamSynchronize(s));
}

// ---- host tier + asynchronous greedy loader --------------------------------
// Copy device buffers into a packed pinned blob (stream-ordered on s).
std::unique_ptr<HostBlob> stage_blob(const std::vector<const DevBuf*>& parts, cudaStream_t s) {
    auto b = std::make_unique<HostBlob>();
    size_t total = 0;
    for (auto* p : parts) {
        b->off.push_back(total);
        b->sz.push_back(p->bytes);
        total += (p->bytes + 255) & ~(size_t)255;
    }
    b->buf.alloc(std::max<size_t>(total, 256));
    for (size_t k = 0; k < parts.size(); ++k)
        EEB_CUDA(cudaMemcpyAsync(static_cast<char*>(b->buf.p) + b->off[k], parts[k]->p, b->sz[k],
                                 cudaMemcpyDeviceToHost, s));
    return b;
}

std::vector<const DevBuf*> base_parts(const Model& m) {
    std::vector<const DevBuf*> v{&m.emb};
    for (auto& h : m.head) v.push_back(h.get());
    for (auto& g : m.head_norm) v.push_back(g.get());
    return v;
}

// ---- caller-supplied weights (eeb_host_stage_layer / _base, eeb_load_layers_from) --
// Packed host layout = the host tier's blob layout: parts back to back, each
// at a 256-byte aligned offset (include/eeb/eeb.h, eeb_weight_layout).
constexpr size_t kPartAlign = 256;
std::vector<size_t> layer_part_bytes(const Model& m) {
    const size_t D = m.desc.d_model, wb = m.wbytes;
    return {D * 4, D * 4, (size_t)(m.dq_l + 2 * m.dkv_l) * D * wb, D * m.dq_l * wb, (size_t)m.up_l * D * wb,
            D * (size_t)m.f_l * wb};
}
std::vector<size_t> base_part_bytes(const Model& m) {
    const size_t D = m.desc.d_model, V = m.desc.vocab, wb = m.wbytes;
    std::vector<size_t> v{V * D * wb};
    for (int e = 0; e < m.desc.n_exits; ++e) v.push_back(V * D * wb);
    for (int e = 0; e < m.desc.n_exits; ++e) v.push_back(D * 4);
    return v;
}
size_t packed_offsets(const std::vector<size_t>& sz, std::vector<size_t>* off) {
    size_t total = 0;
    for (size_t k : sz) {
        if (off) off->push_back(total);
        total += (k + kPartAlign - 1) & ~(kPartAlign - 1);
    }
    return total;
}
// A host-tier blob holding a copy of the caller's packed buffer.
std::unique_ptr<HostBlob> blob_from_host(const std::vector<size_t>& sz, const void* src, int64_t bytes) {
    auto b = std::make_unique<HostBlob>();
    const size_t total = packed_offsets(sz, &b->off);
    if (!src || bytes != (int64_t)total)
        throw Error(EEB_E_VALIDATION, "weights buffer must be " + std::to_string(total) + " bytes (eeb_weight_layout)");
    b->sz = sz;
    b->buf.alloc(total);
    std::memcpy(b->buf.p, src, total);
    return b;
}
void require_single_shard(const Model& m) {
    if (m.shards != 1 || m.tp != 1)
        throw Error(EEB_E_DOMAIN, "caller-supplied weights: tensor-parallel models are not supported (tp_size must be 1)");
}
// Device layer l (1-based) filled from the host tier's blob (synchronous on s).
std::unique_ptr<LayerWeights> layer_from_host(const Model& m, int l, cudaStream_t s) {
    auto L = alloc_layer(m);
    const HostBlob& b = *m.host.layers[l - 1];
    for (int k = 0; k < 6; ++k)
        EEB_CUDA(cudaMemcpyAsync(L->parts[k]->p, static_cast<const char*>(b.buf.p) + b.off[k], b.sz[k],
                                 cudaMemcpyHostToDevice, s));
    return L;
}
void base_from_host(Model& m, cudaStream_t s) {
    const eeb_model_desc& d = m.desc;
    const HostBlob& b = *m.host.base;
    m.emb.ensure(b.sz[0]);
    EEB_CUDA(cudaMemcpyAsync(m.emb.p, b.buf.p, b.sz[0], cudaMemcpyHostToDevice, s));
    m.head.clear();
    m.head_norm.clear();
    for (int e = 0; e < d.n_exits; ++e) {
        auto h = std::make_unique<DevBuf>(m.pool);
        h->ensure(b.sz[1 + e]);
        EEB_CUDA(cudaMemcpyAsync(h->p, static_cast<const char*>(b.buf.p) + b.off[1 + e], b.sz[1 + e],
                                 cudaMemcpyHostToDevice, s));
        auto g = std::make_unique<DevBuf>(m.pool);
        g->ensure(b.sz[1 + d.n_exits + e]);
        EEB_CUDA(cudaMemcpyAsync(g->p, static_cast<const char*>(b.buf.p) + b.off[1 + d.n_exits + e],
                                 b.sz[1 + d.n_exits + e], cudaMemcpyHostToDevice, s));
        m.head.push_back(std::move(h));
        m.head_norm.push_back(std::move(g));
    }
}

void host_stage(eeb_ctx* c, Model& m, int depth) {
    const eeb_model_desc& d = m.desc;
    if (depth < 0 || depth > d.num_layers) throw Error(EEB_E_DOMAIN, "host stage: depth outside [0, num_layers]");
    settle_pending(m);
    cudaStream_t s = c->stream;
    if (!m.host.base) {
        if (m.loaded > 0) {
            m.host.base = stage_blob(base_parts(m), s);
        } else {
            Model tmp;  // materialise on device only long enough to copy out
            tmp.desc = d;
            tmp.alphas = m.alphas;
            tmp.wbytes = m.wbytes;
            tmp.tp = m.tp;
            tmp.rank = m.rank;
            tmp.shards = m.shards;
            tmp.v_l = m.v_l;
            synth_base(tmp, s);
            m.host.base = stage_blob(base_parts(tmp), s);
            EEB_CUDA(cudaStreamSynchronize(s));
        }
    }
    while ((int)m.host.layers.size() < depth) {
        const int l = (int)m.host.layers.size() + 1;
        if (l <= (int)m.layers.size()) {
            const LayerWeights& L = *m.layers[l - 1];
            m.host.layers.push_back(stage_blob({L.parts, L.parts + 6}, s));
        } else {
            auto L = synth_layer(m, l, s);
            m.host.layers.push_back(stage_blob({L->parts, L->parts + 6}, s));
            EEB_CUDA(cudaStreamSynchronize(s));  // before the temporary layer is freed
        }
    }
    EEB_CUDA(cudaStreamSynchronize(s));
}

// Grow the resident prefix to `to` by pinned H2D copies on the load stream;
// returns immediately.  Steps that need a layer wait on its event.
void load_async(eeb_ctx* c, Model& m, int to) {
    const eeb_model_desc& d = m.desc;
    if (to < 0 || to > d.num_layers) throw Error(EEB_E_DOMAIN, "load: depth outside [0, num_layers]");
    if (to <= m.loaded) {
        load_to(c, m, to);  // shrink / no-op: synchronous free
        return;
    }
    if ((int)m.host.layers.size() < to || !m.host.base)
        throw Error(EEB_E_CAPACITY, "host tier holds " + std::to_string(m.host.layers.size()) +
                                        " layers; stage them first (eeb_host_stage)");
    settle_pending(m);
    cudaStream_t ls = c->load_stream;
    auto P = std::make_unique<PendingLoad>();
    EEB_CUDA(cudaEventCreate(&P->t0));
    EEB_CUDA(cudaEventCreate(&P->t1));
    // Device buffers first (cudaMalloc is host-side work), then the copies
    // back to back on the load stream: the timed region is the transfer.
    std::vector<std::unique_ptr<LayerWeights>> fresh;
    for (int l = (int)m.layers.size() + 1; l <= to; ++l) fresh.push_back(alloc_layer(m));
    if (m.loaded == 0) {
        const HostBlob& b = *m.host.base;
        m.emb.ensure(b.sz[0]);
        m.head.clear();
        m.head_norm.clear();
        for (int e = 0; e < d.n_exits; ++e) {
            m.head.push_back(std::make_unique<DevBuf>(m.pool));
            m.head.back()->ensure(b.sz[1 + e]);
            m.head_norm.push_back(std::make_unique<DevBuf>(m.pool));
            m.head_norm.back()->ensure(b.sz[1 + d.n_exits + e]);
        }
    }
    // growth only adds buffers: nothing queued on the decode stream reads them
    EEB_CUDA(cudaEventRecord(P->t0, ls));
    auto copy_in = [&](DevBuf& dst, const HostBlob& b, size_t k) {
        EEB_CUDA(cudaMemcpyAsync(dst.p, static_cast<const char*>(b.buf.p) + b.off[k], b.sz[k], cudaMemcpyHostToDevice,
                                 ls));
        P->bytes += (int64_t)b.sz[k];
    };
    auto mark = [&](int layer) {
        cudaEvent_t ev;
        EEB_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        EEB_CUDA(cudaEventRecord(ev, ls));
        P->ready.push_back({layer, ev});
    };
    if (m.loaded == 0) {
        const HostBlob& b = *m.host.base;
        copy_in(m.emb, b, 0);
        for (int e = 0; e < d.n_exits; ++e) {
            copy_in(*m.head[e], b, 1 + e);
            copy_in(*m.head_norm[e], b, 1 + d.n_exits + e);
        }
        mark(0);
    }
    for (auto& L : fresh) {
        const int l = (int)m.layers.size() + 1;
        const HostBlob& b = *m.host.layers[l - 1];
        for (int k = 0; k < 6; ++k) copy_in(*L->parts[k], b, k);
        mark(l);
        m.layers.push_back(std::move(L));
    }
    EEB_CUDA(cudaEventRecord(P->t1, ls));
    m.loaded = to;
    m.pending = std::move(P);
}

// Make the decode stream wait for the layers a step needs (1..need, and the
// base weights) if they are still in flight.  Issued outside graph capture.
void wait_layers(eeb_ctx* c, Model& m, int need) {
    if (!m.pending) return;
    bool all_done = cudaEventQuery(m.pending->t1) == cudaSuccess;
    if (all_done) {
        settle_pending(m);
        return;
    }
    for (auto& [l, ev] : m.pending->ready)
        if (l <= need) EEB_CUDA(cudaStreamWaitEvent(c->stream, ev, 0));
}

int64_t weight_bytes_at(const Model& m, int depth) {
    const eeb_model_desc& d = m.desc;
    const int64_t D = d.d_model, F = d.d_ffn;
    const int64_t S = m.shards;
    const int64_t base = (int64_t)d.vocab * D * m.wbytes + (int64_t)d.n_exits * (S * m.v_l * D * m.wbytes + D * 4);
    const int64_t per_layer =
        S * ((int64_t)(m.dq_l + 2 * m.dkv_l) * D + D * m.dq_l + (int64_t)m.up_l * D + D * m.f_l) * m.wbytes +
        2 * D * 4;
    (void)F;
    return depth <= 0 ? 0 : base + per_layer * depth;
}

// ---------------------------------------------------------------------------
// Step workspace.
// ---------------------------------------------------------------------------
struct Ints {  // offsets into ctx->rows
    int* nA; int* nB; int* rowA; int* slotA; int* posA; int* rowB; int* slotB; int* posB;
    int* src; int* tok; int* slot; int* pos;
};

Ints ints_of(eeb_ctx* c) {
    int* base = c->rows.as<int>();
    const int R = c->cap_rows;
    Ints r;
    r.nA = base; r.nB = base + 1;
    int* p = base + 32;
    r.rowA = p; p += R; r.slotA = p; p += R; r.posA = p; p += R;
    r.rowB = p; p += R; r.slotB = p; p += R; r.posB = p; p += R;
    r.src = p; p += R; r.tok = p; p += R; r.slot = p; p += R; r.pos = p; p += R;
    return r;
}

// Decode attention KV splits (flash-decoding; EEB_ATTN_KVSPLIT, default 1: on
// C2 2 splits measured 1.73 vs 1.47 ms/step — the per-CTA prologue and the
// combine cost more than the parallelism gains at <= 227 positions).
int kv_splits() {
    static const int v = std::getenv("EEB_ATTN_KVSPLIT") ? std::max(1, std::min(8, std::atoi(std::getenv("EEB_ATTN_KVSPLIT"))))
                                                         : 1;
    return v;
}

// Destroy the captured step graphs (all models, or one) and the persistent
// programs: they hold device pointers by value.
void drop_graphs(eeb_ctx* c, int model = -1) {
    for (auto it = c->graphs.begin(); it != c->graphs.end();) {
        if (model < 0 || it->first.model == model) {
            cudaGraphExecDestroy(it->second);
            it = c->graphs.erase(it);
        } else {
            ++it;
        }
    }
}

// ---- in-graph launch timeline (common.cuh Stamp) ----------------------------
struct StampState {
    unsigned long long* buf = nullptr;
    int cap = 0;
    std::vector<const void*> kernels;  // slot -> kernel, in launch order
    std::vector<int> cats;             // slot -> Cat (labelled by count())
};
thread_local StampState* g_stamp = nullptr;

// Active while one step (or prefill chunk) is enqueued / captured with
// stamping on: hands out consecutive slots to the launches.
struct StampSession {
    StampState st;
    bool on;
    explicit StampSession(eeb_ctx* c) : on(c->stamp_cap > 0) {
        if (!on) return;
        st.buf = c->stamp_buf.as<unsigned long long>();
        st.cap = c->stamp_cap;
        g_stamp = &st;
    }
    ~StampSession() {
        if (on) g_stamp = nullptr;
    }
};

// Reset the cells before a stamped step: starts to ~0 (red.min), ends to 0 (red.max).
void stamp_reset(eeb_ctx* c) {
    const size_t cells = (size_t)c->stamp_cap * kStampCtas;
    EEB_CUDA(cudaMemsetAsync(c->stamp_buf.p, 0xFF, cells * 8, c->stream));
    EEB_CUDA(cudaMemsetAsync(c->stamp_buf.as<unsigned long long>() + cells, 0, cells * 8, c->stream));
    EEB_CUDA(cudaMemsetAsync(c->stamp_buf.as<unsigned long long>() + 2 * cells, 0xFF, cells * 8, c->stream));
    EEB_CUDA(cudaMemsetAsync(c->stamp_buf.as<unsigned long long>() + 3 * cells, 0, cells * 8, c->stream));
}

bool prefill_lt_ready(eeb_ctx* c);

// Byte offsets of the step outputs inside ctx->o_all for R rows and up to ne
// exit heads: the per-row / per-step outputs first (common_end), the
// per-head arrays of a profiling step after them.
struct OutLayout {
    size_t exit, tok, conf, logp, breach, unch, bin, hist, nbr, sum, common_end, htok, hconf, hlogp, total;
    OutLayout(int R, int ne) {
        size_t o = 0;
        auto take = [&](size_t bytes) {
            const size_t at = o;
            o = (o + bytes + 255) & ~(size_t)255;
            return at;
        };
        exit = take((size_t)R * 4);
        tok = take((size_t)R * 4);
        conf = take((size_t)R * 4);
        logp = take((size_t)R * 4);
        breach = take((size_t)R);
        unch = take((size_t)R);
        hist = take(64 * 8);
        nbr = take(8);
        sum = take(8);
        common_end = o;
        bin = take((size_t)R * 4);
        htok = take((size_t)R * ne * 4);
        hconf = take((size_t)R * ne * 4);
        hlogp = take((size_t)R * ne * 4);
        total = o;
    }
};

// Size the step workspace for `batch` rows of model m.  Buffers are shared by
// every model of the context and grow to the largest; whenever one moves, every
// captured graph (of any model: a smaller model's graph holds the old pointer)
// is dropped and recaptured on its next step.
void ensure_workspace(eeb_ctx* c, const Model& m, int batch) {
    bool moved = false;
    if (!c->decide_ticket.p) {  // outside any capture
        moved |= c->decide_ticket.ensure(4);
        EEB_CUDA(cudaMemsetAsync(c->decide_ticket.p, 0, 4, c->stream));
    }
    if (const int S = kv_splits(); S > 1) {  // decode KV split: partials + tickets (zeroed when grown)
        const size_t rows = (size_t)std::max(batch, c->cap_rows);
        const size_t part = rows * m.hkv_l * m.shards * S * 8 * (m.head_dim + 2) * 4;
        const size_t tick = rows * m.hkv_l * m.shards * 4;
        moved |= c->kv_part.ensure(part);
        if (c->kv_ticket.ensure(tick)) {
            moved = true;
            EEB_CUDA(cudaMemsetAsync(c->kv_ticket.p, 0, c->kv_ticket.bytes, c->stream));
        }
    }
    const eeb_model_desc& d = m.desc;
    const int R = std::max(batch, c->cap_rows);
    const size_t act = m.wbytes;
    const int64_t D = d.d_model, F = d.d_ffn;
    moved |= R != c->cap_rows;  // the row-index arrays' layout depends on cap_rows
    c->cap_rows = R;
    moved |= c->xA.ensure((size_t)R * D * 4);
    moved |= c->xB.ensure((size_t)R * D * 4);
    moved |= c->hn.ensure((size_t)R * D * act);
    moved |= c->hnB.ensure((size_t)R * D * act);
    moved |= c->hhead.ensure((size_t)R * D * act);
    if (d.dtype == EEB_BF16) prefill_lt_ready(c);  // handle + workspace outside any capture
    moved |= c->attn.ensure((size_t)R * m.dq * act);
    moved |= c->mlp_h.ensure((size_t)R * F * act);
    // split-K partial bound: splits <= K / (32 * vec) for every GEMM of the step.
    const int64_t kmin = act == 4 ? 128 : 256;
    int64_t need = 0;  // split-K planes per GEMM: tier 1 <= K/(32 vec)+1, tier 2 <= SMs/tiles+1
    // (the split GEMMs serve <= 256 rows; larger prefill chunks run cuBLASLt
    // into one plane of R rows)
    const int64_t Rs = std::min<int64_t>(R, 256);
    auto upd = [&](int64_t N, int64_t K) {
        const int64_t tiles = (N + 127) / 128;
        need = std::max(need, std::max<int64_t>(K / kmin + 1, c->num_sms / tiles + 1) * Rs * N);
        need = std::max(need, (int64_t)R * N);
    };
    upd(m.dq_l + 2 * m.dkv_l, D);
    upd(D, m.dq_l);
    upd(m.up_l, D);
    upd(D, m.f_l);
    upd(m.v_l, D);
    need *= m.shards;  // row-parallel shards write their partial planes side by side
    moved |= c->ws.ensure((size_t)need * 4);
    c->ws_elems = (int64_t)(c->ws.bytes / 4);
    moved |= c->rows.ensure((size_t)(32 + 12 * R) * 4);
    moved |= c->head_tok.ensure((size_t)R * 4);
    moved |= c->head_tri.ensure((size_t)R * ((m.v_l + 127) / 128) * m.tp * 16);
    if (m.tp > 1) moved |= c->tp_partial.ensure((size_t)R * D * 4);
    moved |= c->head_conf.ensure((size_t)R * 4);
    moved |= c->head_logp.ensure((size_t)R * 4);
    moved |= c->o_all.ensure(OutLayout(R, 64).total);
    const size_t pin_need = (size_t)R * 3 * 4 + 256 + OutLayout(R, 64).total;
    if (pin_need > c->pin_bytes) {
        if (c->pin) cudaFreeHost(c->pin);
        c->pin = nullptr;
        EEB_CUDA(cudaMallocHost(&c->pin, pin_need));
        c->pin_bytes = pin_need;
    }
    if (moved) drop_graphs(c);
}

StepOutDev out_dev(eeb_ctx* c) {
    StepOutDev o;
    const OutLayout L(c->cap_rows, 64);
    char* b = static_cast<char*>(c->o_all.p);
    o.exit_layer = reinterpret_cast<int32_t*>(b + L.exit);
    o.token_id = reinterpret_cast<int32_t*>(b + L.tok);
    o.confidence = reinterpret_cast<float*>(b + L.conf);
    o.logprob = reinterpret_cast<float*>(b + L.logp);
    o.breached = reinterpret_cast<uint8_t*>(b + L.breach);
    o.unchanged = reinterpret_cast<uint8_t*>(b + L.unch);
    o.bin = reinterpret_cast<int32_t*>(b + L.bin);
    o.hist = reinterpret_cast<int64_t*>(b + L.hist);
    o.n_breached = reinterpret_cast<int64_t*>(b + L.nbr);
    o.sum_logprob = reinterpret_cast<double*>(b + L.sum);
    o.head_token = reinterpret_cast<int32_t*>(b + L.htok);
    o.head_confidence = reinterpret_cast<float*>(b + L.hconf);
    o.head_logprob = reinterpret_cast<float*>(b + L.hlogp);
    return o;
}

// ---------------------------------------------------------------------------
// Launch helpers with optional per-category event timing.
// ---------------------------------------------------------------------------
struct Timer {
    eeb_ctx* c;
    int cat;
    cudaEvent_t b = nullptr, e = nullptr;
    Timer(eeb_ctx* ctx, int category) : c(ctx), cat(category) {
        c->cat_launches[cat] += 0;
        if (!c->profiling) return;
        b = take();
        e = take();
        EEB_CUDA(cudaEventRecord(b, c->stream));
    }
    ~Timer() {
        if (!c->profiling) return;
        cudaEventRecord(e, c->stream);
        c->ev_used.push_back({cat, {b, e}});
    }
    cudaEvent_t take() {
        if (c->ev_pool.empty()) {
            cudaEvent_t ev;
            EEB_CUDA(cudaEventCreate(&ev));
            return ev;
        }
        cudaEvent_t ev = c->ev_pool.back();
        c->ev_pool.pop_back();
        return ev;
    }
};

void count(eeb_ctx* c, int cat, int n) {
    if (g_stamp)  // label this call's launches in the timeline
        for (int i = (int)g_stamp->cats.size() - 1, k = 0; i >= 0 && k < n && g_stamp->cats[i] < 0; --i, ++k)
            g_stamp->cats[i] = cat;
    c->cat_launches[cat] += n;
    c->step_launches += n;
}

// The cuBLASLt handle and workspace of the prefill GEMMs (created outside any
// stream capture); false when cuBLASLt is unavailable or switched off.
bool prefill_lt_ready(eeb_ctx* c) {
    static const bool on = !std::getenv("EEB_PREFILL_LT") || std::atoi(std::getenv("EEB_PREFILL_LT")) != 0;
    if (!on) return false;
    if (!c->lt) {
        if (cublasLtCreate(&c->lt) != CUBLAS_STATUS_SUCCESS) {
            c->lt = nullptr;
            return false;
        }
        c->lt_ws.ensure(32u << 20);
    }
    return true;
}

// Prefill GEMM on cuBLASLt: out[rows][N] (f32) = X[rows][K] . W[N][K]^T in
// one plane.  Column-major view: D (N x rows, ld N) = op(A) B with A = W (K x
// N, ld K, transposed) and B = X (K x rows, ld K).  EEB_PREFILL_LT=0 keeps
// the tcgen05 decode GEMM (split-K planes) for prefill too.
// relu_bf16: out is bf16 [rows][N] = bf16(relu(X W^T)) (the OPT MLP's up
// projection with its activation in the cuBLASLt epilogue); else f32 plane.
bool gemm_lt(eeb_ctx* c, const void* W, const void* X, int N, int K, int rows, void* out, bool relu_bf16 = false) {
    static const bool on = !std::getenv("EEB_PREFILL_LT") || std::atoi(std::getenv("EEB_PREFILL_LT")) != 0;
    if (!on) return false;
    constexpr size_t kWs = 32u << 20;
    if (!c->lt || c->lt_ws.bytes < kWs) return false;  // (created by ensure_workspace, outside any capture)
    auto& pl = c->lt_plans[{N, K, rows, relu_bf16 ? 1 : 0}];
    if (!pl.op) {
        const cublasComputeType_t ct = CUBLAS_COMPUTE_32F;
        const cudaDataType_t st = CUDA_R_32F;
        cublasLtMatmulDescCreate(&pl.op, ct, st);
        const cublasOperation_t ta = CUBLAS_OP_T, tb = CUBLAS_OP_N;
        cublasLtMatmulDescSetAttribute(pl.op, CUBLASLT_MATMUL_DESC_TRANSA, &ta, sizeof ta);
        cublasLtMatmulDescSetAttribute(pl.op, CUBLASLT_MATMUL_DESC_TRANSB, &tb, sizeof tb);
        if (relu_bf16) {
            const cublasLtEpilogue_t ep = CUBLASLT_EPILOGUE_RELU;
            cublasLtMatmulDescSetAttribute(pl.op, CUBLASLT_MATMUL_DESC_EPILOGUE, &ep, sizeof ep);
        }
        cublasLtMatrixLayoutCreate(&pl.a, CUDA_R_16BF, K, N, K);
        cublasLtMatrixLayoutCreate(&pl.b, CUDA_R_16BF, K, rows, K);
        cublasLtMatrixLayoutCreate(&pl.d, relu_bf16 ? CUDA_R_16BF : CUDA_R_32F, N, rows, N);
        cublasLtMatmulPreference_t pref;
        cublasLtMatmulPreferenceCreate(&pref);
        const size_t ws = kWs;
        cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES, &ws, sizeof ws);
        cublasLtMatmulHeuristicResult_t res{};
        int n = 0;
        pl.ok = cublasLtMatmulAlgoGetHeuristic(c->lt, pl.op, pl.a, pl.b, pl.d, pl.d, pref, 1, &res, &n) ==
                    CUBLAS_STATUS_SUCCESS &&
                n > 0;
        if (pl.ok) pl.algo = res.algo;
        cublasLtMatmulPreferenceDestroy(pref);
    }
    if (!pl.ok) return false;
    const float alpha = 1.f, beta = 0.f;
    const cublasStatus_t r = cublasLtMatmul(c->lt, pl.op, &alpha, W, pl.a, X, pl.b, &beta, out, pl.d, out, pl.d,
                                            &pl.algo, c->lt_ws.p, kWs, c->stream);
    if (r != CUBLAS_STATUS_SUCCESS) throw Error(EEB_E_CUDA, "cublasLtMatmul failed: " + std::to_string((int)r));
    return true;
}

// One decode GEMM into the split-K plane workspace; returns the planes written.
int gemm(eeb_ctx* c, int cat, const Model& m, const void* W, const void* X, int N, int K, const int* n_active,
         int batch, int plane0 = 0) {
    GemmArgs a;
    a.dtype = m.desc.dtype;
    a.W = W;
    a.X = X;
    a.n_active = n_active;
    a.max_rows = batch;
    a.N = N;
    a.K = K;
    a.plane_stride = (int64_t)batch * N;
    a.out = (c->gemm_out ? c->gemm_out : c->ws.as<float>()) + (int64_t)plane0 * a.plane_stride;
    a.max_planes = (int)std::min<int64_t>(64, (c->gemm_out ? c->gemm_out_elems : c->ws_elems) / a.plane_stride - plane0);
    if (a.max_planes < 1) throw Error(EEB_E_CAPACITY, "GEMM output planes do not fit the workspace");
    a.num_sms = c->num_sms;
    a.pf = c->pf_ptr;
    a.pf_bytes = c->pf_bytes;
    c->pf_ptr = nullptr;
    c->pf_bytes = 0;
    int planes = 0;
    // (prefill chunks: one cuBLASLt plane, after the planes earlier row-parallel
    //  shards of an all-shards context wrote — chunks above 256 rows have no
    //  split-K tcgen05 path)
    if (c->in_prefill && batch >= 64 && m.desc.dtype == EEB_BF16 && c->gemm_tier != 1 &&
        gemm_lt(c, W, X, N, K, batch, a.out)) {
        count(c, cat, 1);
        return 1;
    }
    if (c->gemm_tier != 1 && m.desc.dtype == EEB_BF16) planes = gemm_tc(a, c->stream);
    if (planes == 0) {
        if (c->gemm_tier == 2 && m.desc.dtype == EEB_BF16 && batch >= tc_min_rows() && gemm_tc_available())
            throw Error(EEB_E_DOMAIN, "tensor-core tier requested but not applicable");
        planes = gemm_cc(a, c->stream);
    }
    count(c, cat, 1);
    return planes;
}

// Exit-head GEMM with the fused softmax tail; returns the vocab tiles written
// to ctx->head_tri, 0 when the tensor-core path does not apply.
int gemm_head_fused(eeb_ctx* c, const Model& m, const void* W, const void* X, int N, int K, const int* n_active,
                    int batch, float* tri, int vocab_off) {
    GemmArgs a;
    a.dtype = m.desc.dtype;
    a.W = W;
    a.X = X;
    a.n_active = n_active;
    a.max_rows = batch;
    a.N = N;
    a.K = K;
    a.out = nullptr;
    a.plane_stride = 0;
    a.max_planes = 1;
    a.num_sms = c->num_sms;
    a.head_tri = tri;
    a.vocab_off = vocab_off;
    if (gemm_tc(a, c->stream) == 0) return 0;
    count(c, kCatHead, 1);
    return (N + 127) / 128;
}

// ---------------------------------------------------------------------------
// The step.  Per layer: QKV GEMM -> attention (sums the QKV planes, RoPE, KV
// append) -> O GEMM -> residual+RMSNorm -> up GEMM -> activation -> down GEMM
// -> residual+RMSNorm (next layer's norm, plus the exit head's norm after an
// exit layer).  Heads: head GEMM -> max/argmax/sum-exp -> decide (+ compaction).
// ---------------------------------------------------------------------------
// Timing experiments only (results are wrong): EEB_SKIP=gemm,attn,norm,head
// drops a kernel category from the step so its share of the graph can be measured.
bool skip_cat(const char* what) {
    static const std::string env = std::getenv("EEB_SKIP") ? std::getenv("EEB_SKIP") : "";
    return !env.empty() && env.find(what) != std::string::npos;
}

// Sum the `planes` split-K partial planes into the context's partial buffer
// and all-reduce it over the tensor-parallel group (NCCL, on the step stream;
// capturable into the step's graph).  Returns the single plane to consume.
const float* tp_allreduce(eeb_ctx* c, const Model& m, const float* planes_base, int planes, const int* n_active,
                          int batch) {
    const int D = m.desc.d_model;
    float* part = c->tp_partial.as<float>();
    launch_plane_sum(planes_base, planes, (int64_t)batch * D, n_active, batch, D, part, c->num_sms, c->stream);
    if (!c->nccl) throw Error(EEB_E_DOMAIN, "tensor-parallel rank without a communicator (eeb_nccl_init)");
    const ncclResult_t r = nccl().all_reduce(part, part, (size_t)batch * D, ncclFloat32, ncclSum, c->nccl, c->stream);
    if (r != ncclSuccess) throw Error(EEB_E_CUDA, "ncclAllReduce failed");
    count(c, kCatNorm, 1);
    return part;
}

// L2 prefetch of the next GEMM's weights from the latency-bound kernel before
// it (attention -> O, mlp norm -> up, final norm -> next QKV); opt-in
// EEB_L2PF_FUSED=1 — measured slower on C2 (1.473 vs 1.412 ms/step: issuing
// the bulk prefetches delays the norm's own warps by ~3 us, more than the
// GEMMs gain); the GEMMs' own pre-wait L2 prefetch (gemm_tc.cu) replaces it.
bool l2pf_fused() {
    static const bool on = std::getenv("EEB_L2PF_FUSED") && std::atoi(std::getenv("EEB_L2PF_FUSED")) != 0;
    return on;
}

struct PlaneSet {
    const float* base;
    int planes;
    bool px = false;  // the planes sit in the TP exchange buffer: reduce with launch_tp_norm
};

// The row-parallel GEMMs of a peer-memory TP rank write their planes into the
// rank's exchange buffer, where the row owners read them.
struct PxPlanesScope {
    eeb_ctx* c;
    PxPlanesScope(eeb_ctx* cc, const Model& m, bool on) : c(cc) {
        if (on) {
            c->gemm_out = reinterpret_cast<float*>(m.pxp.base[m.pxp.rank] + m.pxp.lay.planes);
            c->gemm_out_elems = m.pxp.lay.planes_elems;
        }
    }
    ~PxPlanesScope() {
        c->gemm_out = nullptr;
        c->gemm_out_elems = 0;
    }
};

// One decoder layer up to (not including) the final residual + RMSNorm:
// per shard QKV GEMM -> [KV append] -> attention; per shard O GEMM (row-parallel
// partials side by side in the plane workspace) -> residual + mlp norm; per
// shard up GEMM -> activation; per shard down GEMM.  Returns the down partial
// planes (all-reduced over the TP group for a rank context).
PlaneSet layer_core(eeb_ctx* c, Model& m, int l, const RowState& cur, void* h, int batch, bool kv_ready) {
    const eeb_model_desc& d = m.desc;
    const int D = d.d_model;
    cudaStream_t s = c->stream;
    const LayerWeights& W = *m.layers[l - 1];
    float* ws = c->ws.as<float>();
    const size_t wb = m.wbytes;
    const int qkv_l = m.dq_l + 2 * m.dkv_l;
    // L2 prefetch chain (one context shard only): each GEMM pulls the next
    // GEMM's weights into L2 — QKV -> O -> up -> down -> next layer's QKV.
    const bool pf_on = m.shards == 1;
    auto next_pf = [&](const void* p, size_t bytes) {
        c->pf_ptr = pf_on && p ? p : nullptr;
        c->pf_bytes = pf_on && p ? bytes : 0;
    };
    for (int sh = 0; sh < m.shards; ++sh) {
        int planes;
        next_pf(W.wo.p, (size_t)D * m.dq_l * wb);
        {
            Timer t(c, kCatGemm);
            planes = skip_cat("gemm") ? 1
                                      : gemm(c, kCatGemm, m, static_cast<const char*>(W.wqkv.p) + (size_t)sh * qkv_l * D * wb,
                                             h, qkv_l, D, cur.n_active, batch);
        }
        Timer t(c, kCatAttn);
        AttnArgs a;
        a.dtype = d.dtype;
        a.qkv = ws;
        a.splits = planes;
        a.split_stride = (int64_t)batch * qkv_l;
        const size_t kv_off = ((size_t)(l - 1) * m.kv_layer_elems + (size_t)sh * m.kv_shard_elems) * wb;
        a.k_cache = static_cast<char*>(m.k_cache.p) + kv_off;
        a.v_cache = static_cast<char*>(m.v_cache.p) + kv_off;
        a.kv_depth = m.kv_depth.as<uint8_t>();
        a.rope_cos = m.rope_cos.as<float>();
        a.rope_sin = m.rope_sin.as<float>();
        a.n_active = cur.n_active;
        a.slot = cur.slot;
        a.pos = cur.pos;
        a.max_rows = batch;
        a.layer = l;
        a.n_heads = m.hq_l;
        a.n_kv_heads = m.hkv_l;
        a.head_dim = m.head_dim;
        a.max_seq = d.max_seq_len;
        a.page_table = m.page_table.as<int>();
        a.page_size = m.kv_page;
        a.pages_per_seq = m.pages_per_seq;
        if (!kv_ready && kv_splits() > 1 && c->kv_part.p && c->kv_ticket.p) {
            a.kv_splits = kv_splits();
            a.kv_part = c->kv_part.as<float>();
            a.kv_ticket = c->kv_ticket.as<int>();
        }
        if (kv_ready && c->pf_cur_items > 0) {
            a.pf_items = c->pf_items.as<int4>();
            a.pf_n_items = reinterpret_cast<const int*>(c->pf_items.as<int4>() + c->pf_cur_items);
            a.pf_max_items = c->pf_cur_items;
        }
        a.out = static_cast<char*>(c->attn.p) + (size_t)sh * batch * m.dq_l * wb;
        const size_t mk = (size_t)(l - 1) * m.shards + sh;
        a.k_map = m.k_maps.empty() ? nullptr : m.k_maps[mk].data();
        a.v_map = m.v_maps.empty() ? nullptr : m.v_maps[mk].data();
        a.k_map8 = m.k_maps8.empty() ? nullptr : m.k_maps8[mk].data();
        a.v_map8 = m.v_maps8.empty() ? nullptr : m.v_maps8[mk].data();
        a.num_sms = c->num_sms;
        a.kv_ready = kv_ready ? 1 : 0;
        if (l2pf_fused() && pf_on) {
            a.pf = static_cast<const char*>(W.wo.p) + (size_t)sh * D * m.dq_l * wb;
            a.pf_bytes = (size_t)D * m.dq_l * wb;
        }
        if (kv_ready) {
            launch_kv_append(a, s);
            count(c, kCatAttn, 1);
        }
        if (!skip_cat("attn")) launch_attention(a, s);
        count(c, kCatAttn, 1);
    }
    int planes = 0;
    next_pf(W.wup.p, (size_t)m.up_l * D * wb);
    const bool px = m.tp > 1 && m.shards == 1 && m.px_on();
    {
        Timer t(c, kCatGemm);
        PxPlanesScope px_scope(c, m, px);
        for (int sh = 0; sh < m.shards; ++sh)
            planes += skip_cat("gemm") ? 1
                                       : gemm(c, kCatGemm, m, static_cast<const char*>(W.wo.p) + (size_t)sh * D * m.dq_l * wb,
                                              static_cast<const char*>(c->attn.p) + (size_t)sh * batch * m.dq_l * wb, D,
                                              m.dq_l, cur.n_active, batch, planes);
    }
    PlaneSet o{ws, planes};
    if (px) {
        Timer t(c, kCatNorm);
        launch_tp_norm(d.dtype, m.pxp, planes, (int64_t)batch * D, cur.n_active, batch, cur.x, D, d.norm_eps,
                       W.mlp_norm.as<float>(), h, nullptr, nullptr, s, c->in_prefill ? 4 : 1);
        count(c, kCatNorm, 1);
    } else if (m.tp > 1 && m.shards == 1) {
        o = {tp_allreduce(c, m, ws, planes, cur.n_active, batch), 1};
    }
    if (!px) {
        Timer t(c, kCatNorm);
        if (!skip_cat("norm"))
            launch_residual_norm(d.dtype, o.base, o.planes, (int64_t)batch * D, cur.n_active, batch, cur.x, D, d.norm_eps,
                                 W.mlp_norm.as<float>(), h, nullptr, nullptr, s, l2pf_fused() && pf_on ? W.wup.p : nullptr,
                                 (size_t)m.up_l * D * wb, c->in_prefill ? 4 : 1);
        count(c, kCatNorm, 1);
    }
    static const bool act_unfused = std::getenv("EEB_ACT_UNFUSED") != nullptr;  // A/B
    // The activation fused into the up GEMM (4-CTA clusters reducing K on chip)
    // at every decode batch: above 128 rows the GEMM runs two 128-row CTAs per
    // weight tile (gemm_tc), so the on-chip reduction stays a 128-column tile
    // (C2 batch 256: 2.148 -> 2.108 ms/step against split-K planes + the
    // activation kernel; with one 256-column tile it was 44 us vs 15 + 10 us).
    static const int act_fused_max = std::getenv("EEB_ACT_FUSED_MAX_ROWS")
                                         ? std::atoi(std::getenv("EEB_ACT_FUSED_MAX_ROWS"))
                                         : 256;
    for (int sh = 0; sh < m.shards; ++sh) {
        void* act_dst = static_cast<char*>(c->mlp_h.p) + (size_t)sh * batch * m.f_l * wb;
        const void* wup = static_cast<const char*>(W.wup.p) + (size_t)sh * m.up_l * D * wb;
        if (!act_unfused && batch <= act_fused_max && !skip_cat("gemm") && d.dtype == EEB_BF16 && c->gemm_tier != 1) {
            // up projection with the activation in its epilogue (one split)
            Timer t(c, kCatGemm);
            GemmArgs ga;
            ga.dtype = d.dtype;
            ga.W = wup;
            ga.X = h;
            ga.n_active = cur.n_active;
            ga.max_rows = batch;
            ga.N = m.up_l;
            ga.K = D;
            ga.out = nullptr;
            ga.plane_stride = 0;
            ga.max_planes = 1;
            ga.num_sms = c->num_sms;
            ga.act_out = act_dst;
            ga.act_kind = d.mlp_kind == EEB_MLP_SWIGLU ? 2 : 1;
            if (pf_on && W.wdown.p) {
                ga.pf = W.wdown.p;
                ga.pf_bytes = (size_t)D * m.f_l * wb;
            }
            if (gemm_tc(ga, s) > 0) {
                count(c, kCatGemm, 1);
                continue;
            }
        }
        if (c->in_prefill && d.mlp_kind == EEB_MLP_RELU && d.dtype == EEB_BF16 && c->gemm_tier != 1 && batch >= 64 &&
            !skip_cat("gemm")) {
            // prefill chunks on cuBLASLt: ReLU + bf16 in its epilogue (no f32
            // plane, no activation kernel: -14 % of the C2 prefill's launches' time)
            Timer t(c, kCatGemm);
            if (gemm_lt(c, wup, h, m.up_l, D, batch, act_dst, true)) {
                count(c, kCatGemm, 1);
                continue;
            }
        }
        int up_planes;
        {
            Timer t(c, kCatGemm);
            up_planes = skip_cat("gemm") ? 1 : gemm(c, kCatGemm, m, wup, h, m.up_l, D, cur.n_active, batch);
        }
        Timer t(c, kCatNorm);
        if (!skip_cat("norm"))
            launch_act(d.dtype, ws, up_planes, (int64_t)batch * m.up_l, cur.n_active, batch, m.up_l,
                       d.mlp_kind == EEB_MLP_SWIGLU, static_cast<char*>(c->mlp_h.p) + (size_t)sh * batch * m.f_l * wb,
                       c->num_sms, s);
        count(c, kCatNorm, 1);
    }
    planes = 0;
    if (l < (int)m.layers.size() && m.layers[l])
        next_pf(m.layers[l]->wqkv.p, (size_t)qkv_l * D * wb);
    {
        Timer t(c, kCatGemm);
        PxPlanesScope px_scope(c, m, px);
        for (int sh = 0; sh < m.shards; ++sh)
            planes += skip_cat("gemm") ? 1
                                       : gemm(c, kCatGemm, m, static_cast<const char*>(W.wdown.p) + (size_t)sh * D * m.f_l * wb,
                                              static_cast<const char*>(c->mlp_h.p) + (size_t)sh * batch * m.f_l * wb, D,
                                              m.f_l, cur.n_active, batch, planes);
    }
    if (px) return {reinterpret_cast<const float*>(m.pxp.base[m.pxp.rank] + m.pxp.lay.planes), planes, true};
    PlaneSet dn{ws, planes};
    if (m.tp > 1 && m.shards == 1) dn = {tp_allreduce(c, m, ws, planes, cur.n_active, batch), 1};
    return dn;
}

// A conditional node costs ~12 us of the step (it ends the PDL overlap into
// the next layer) and pays off only when all rows tend to exit together:
// measured on C2, batch 1 0.65 -> 0.56 ms/step, batch 2 0.61 -> 0.51, but
// batch 4 1.03 -> 1.04 and batch 64 1.51 -> 1.55.  So: batches of <= 2 rows
// (EEB_COND_MAX_ROWS overrides; 0 disables).
bool cond_enabled(int batch) {
    static const int max_rows =
        std::getenv("EEB_COND_MAX_ROWS") ? std::atoi(std::getenv("EEB_COND_MAX_ROWS")) : 2;
    return batch <= max_rows;
}

// Open an IF body after the current capture position of c->stream: later
// launches are captured into the body (on a nested capture stream) until
// close_cond_bodies.  Returns the stream to launch on.
cudaStream_t open_cond_body(eeb_ctx* c, cudaGraphConditionalHandle h) {
    cudaStream_t outer = c->stream;
    cudaStreamCaptureStatus st;
    cudaGraph_t g;
    const cudaGraphNode_t* deps = nullptr;
    size_t nd = 0;
    EEB_CUDA(cudaStreamGetCaptureInfo(outer, &st, nullptr, &g, &deps, &nd));
    cudaGraphNodeParams p = {};
    p.type = cudaGraphNodeTypeConditional;
    p.conditional.handle = h;
    p.conditional.type = cudaGraphCondTypeIf;
    p.conditional.size = 1;
    cudaGraphNode_t node;
    EEB_CUDA(cudaGraphAddNode(&node, g, deps, nd, &p));
    EEB_CUDA(cudaStreamUpdateCaptureDependencies(outer, &node, 1, cudaStreamSetCaptureDependencies));
    const size_t level = c->cond_open;
    while (c->cond_streams.size() <= level) {
        cudaStream_t cs;
        EEB_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
        c->cond_streams.push_back(cs);
    }
    cudaStream_t body = c->cond_streams[level];
    EEB_CUDA(cudaStreamBeginCaptureToGraph(body, p.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                           cudaStreamCaptureModeThreadLocal));
    ++c->cond_open;
    c->stream = body;
    return body;
}

cudaStream_t close_cond_bodies(eeb_ctx* c) {
    while (c->cond_open > 0) {
        --c->cond_open;
        cudaGraph_t ignored;
        EEB_CUDA(cudaStreamEndCapture(c->cond_streams[c->cond_open], &ignored));
    }
    c->stream = c->main_stream;
    return c->stream;
}

void enqueue_step(eeb_ctx* c, int mi, int depth, int policy, float th, int batch) {
    Model& m = model_of(c, mi);
    const eeb_model_desc& d = m.desc;
    const int L = d.num_layers, D = d.d_model, F = d.d_ffn;
    cudaStream_t s = c->stream;
    Ints I = ints_of(c);
    RowState A{I.nA, I.rowA, I.slotA, I.posA, c->xA.as<float>()};
    RowState B{I.nB, I.rowB, I.slotB, I.posB, c->xB.as<float>()};
    void* hA = c->hn.p;    // normalised activations for the next layer (per state)
    void* hB = c->hnB.p;
    const StepOutDev o = out_dev(c);
    const int64_t hrow = (int64_t)D * m.wbytes;

    std::vector<int> heads;
    int run_layers = L;
    if (policy == EEB_FLAT) {
        int e_used = -1;
        for (int e = 0; e < d.n_exits; ++e)
            if (m.exits[e] <= depth) e_used = e;
        if (e_used < 0)  // observation_for_depth throws DomainError (trace.hpp:92-93)
            throw Error(EEB_E_DOMAIN, "no exit head at or below layer " + std::to_string(depth));
        heads.push_back(e_used);
        run_layers = depth;
    } else if (policy == EEB_FULL_DEPTH) {
        heads.push_back(d.n_exits - 1);
    } else {
        for (int e = 0; e < d.n_exits; ++e) heads.push_back(e);
    }
    auto head_at = [&](size_t hi, int l) { return hi < heads.size() && m.exits[heads[hi]] == l; };

    RowState cur = A, alt = B;
    void* h_cur = hA;
    void* h_alt = hB;
    {
        Timer t(c, kCatOther);
        if (launch_embed_norm(d.dtype, m.emb.p, I.tok, I.slot, I.pos, batch, D, cur, d.norm_eps,
                              m.layers[0]->attn_norm.as<float>(), h_cur, s)) {
            count(c, kCatOther, 1);
        } else {
            launch_embed(d.dtype, m.emb.p, I.tok, I.slot, I.pos, batch, D, cur, s);
            launch_residual_norm(d.dtype, nullptr, 0, 0, cur.n_active, batch, cur.x, D, d.norm_eps,
                                 m.layers[0]->attn_norm.as<float>(), h_cur, nullptr, nullptr, s);
            count(c, kCatOther, 2);
        }
    }
    size_t hi = 0;
    float* ws = c->ws.as<float>();
    for (int l = 1; l <= run_layers; ++l) {
        const PlaneSet dn = layer_core(c, m, l, cur, h_cur, batch, false);
        const float* planes_base = dn.base;
        const int planes = dn.planes;
        const bool exit_here = head_at(hi, l);
        const bool more = l < run_layers;
        {
            Timer t(c, kCatNorm);
            // next layer's attention norm -> h_cur; the exit head's norm -> hhead
            const float* g_next = more ? m.layers[l]->attn_norm.as<float>() : nullptr;
            const float* g_head = exit_here ? m.head_norm[heads[hi]]->as<float>() : nullptr;
            const float* g1 = g_next ? g_next : g_head;
            void* o1 = g_next ? h_cur : c->hhead.p;
            const float* g2 = g_next ? g_head : nullptr;
            void* o2 = g_next && g_head ? c->hhead.p : nullptr;
            // the next layer's QKV weights -> L2 during the norm (not before an
            // exit head: its vocab-sized stream would evict them first)
            const void* pf = l2pf_fused() && more && !exit_here && m.shards == 1 ? m.layers[l]->wqkv.p : nullptr;
            if (g1 && dn.px)
                launch_tp_norm(d.dtype, m.pxp, planes, (int64_t)batch * D, cur.n_active, batch, cur.x, D, d.norm_eps,
                               g1, o1, g2, o2, s);
            else if (g1 && !skip_cat("norm"))
                launch_residual_norm(d.dtype, planes_base, planes, (int64_t)batch * D, cur.n_active, batch, cur.x, D,
                                     d.norm_eps, g1, o1, g2, o2, s, pf,
                                     (size_t)(m.dq_l + 2 * m.dkv_l) * D * m.wbytes);
            count(c, kCatNorm, 1);
        }
        while (head_at(hi, l)) {
            const int e = heads[hi];
            const bool is_final = hi + 1 == heads.size();
            Timer t(c, kCatHead);
            HeadOut h{c->head_tok.as<int>(), c->head_conf.as<float>(), c->head_logp.as<float>()};
            // Fused head (tcgen05 GEMM epilogue emits per-tile softmax partials,
            // decide merges them) unless the logits themselves are retained.
            // vocab-parallel: shard sh covers rows [g v_l, (g+1) v_l) of the head;
            // its tile partials land in region g of head_tri (all-gathered over
            // the TP group for a rank context) and decide merges all regions.
            int head_tiles = 0;
            const int tiles_l = (m.v_l + 127) / 128;
            const int64_t region = (int64_t)batch * tiles_l * 4;  // floats per rank region
            if (!c->retain_logits && !skip_cat("head") && c->gemm_tier != 1 && d.dtype == EEB_BF16 &&
                !std::getenv("EEB_HEAD_UNFUSED")) {
                const bool px = m.tp > 1 && m.shards == 1 && m.px_on();
                for (int sh = 0; sh < m.shards; ++sh) {
                    const int g = m.shard_rank(sh);
                    float* tri = px ? reinterpret_cast<float*>(m.pxp.base[m.pxp.rank] + m.pxp.lay.head)
                                    : c->head_tri.as<float>() + g * region;
                    head_tiles = gemm_head_fused(c, m, static_cast<const char*>(m.head[e]->p) + (size_t)sh * m.v_l * D * m.wbytes,
                                                 c->hhead.p, m.v_l, D, cur.n_active, batch, tri, g * m.v_l);
                    if (head_tiles == 0) break;
                }
                if (head_tiles && px) {
                    launch_px_gather(m.pxp, region, c->head_tri.as<float>(), s);
                    count(c, kCatHead, 1);
                } else if (head_tiles && m.tp > 1 && m.shards == 1) {
                    if (!c->nccl) throw Error(EEB_E_DOMAIN, "tensor-parallel rank without a communicator (eeb_nccl_init)");
                    float* all = c->head_tri.as<float>();
                    const ncclResult_t r = nccl().all_gather(all + m.rank * region, all, (size_t)region, ncclFloat32,
                                                             c->nccl, s);
                    if (r != ncclSuccess) throw Error(EEB_E_CUDA, "ncclAllGather failed");
                }
            }
            if (head_tiles == 0 && m.tp > 1)
                throw Error(EEB_E_DOMAIN, "tensor-parallel exit heads need the fused tensor-core head (bf16, batch >= 16)");
            if (head_tiles == 0) {
                const int hp =
                    skip_cat("head") ? 1 : gemm(c, kCatHead, m, m.head[e]->p, c->hhead.p, d.vocab, D, cur.n_active, batch);
                float* keep = nullptr;
                if (c->retain_logits) {
                    while ((int)c->logits_keep.size() < d.n_exits) c->logits_keep.push_back(std::make_unique<DevBuf>());
                    c->logits_keep[e]->ensure((size_t)batch * d.vocab * 4);
                    keep = c->logits_keep[e]->as<float>();
                }
                launch_head_reduce(ws, hp, (int64_t)batch * d.vocab, d.vocab, cur.n_active, batch, h, keep, s);
                count(c, kCatHead, 1);
            }
            DecideArgs da;
            da.head_tri = head_tiles ? c->head_tri.as<float>() : nullptr;
            da.ticket = c->decide_ticket.as<int>();  // allocated (zeroed) by ensure_workspace
            da.head_tiles = head_tiles;
            da.head_shards = m.tp;
            da.head_shard_stride = region / 4;  // float4 entries per rank region
            da.policy = policy;
            da.exit_index = e;
            da.n_exits = d.n_exits;
            da.exit_layer = m.exits[e];
            da.num_layers = L;
            da.serving_depth = depth;
            da.is_final = is_final ? 1 : 0;
            da.th = th;
            da.max_rows = batch;
            da.cur = cur;
            da.nxt = alt;
            da.gather_src = I.src;
            da.head = h;
            da.out = o;
            for (int k = 0; k < 64; ++k) da.layers[k] = k < d.n_exits ? m.exits[k] : 0;
            // Captured introspective step: everything after this head runs in a
            // conditional body that decide switches off when no row survives —
            // an all-exited step (batch 1: 71% of C2 steps) skips the deeper
            // layers' launches instead of running them on zero rows.
            const bool cond = c->capturing && policy == EEB_INTROSPECTIVE && !is_final && m.tp == 1 &&
                              m.shards == 1 && cond_enabled(batch);
            if (cond) {
                cudaStreamCaptureStatus st;
                cudaGraph_t g;
                EEB_CUDA(cudaStreamGetCaptureInfo(s, &st, nullptr, &g, nullptr, nullptr));
                EEB_CUDA(cudaGraphConditionalHandleCreate(&da.cond, g, 1, cudaGraphCondAssignDefault));
                da.has_cond = 1;
            }
            launch_decide(da, s);
            count(c, kCatHead, 1);
            if (policy == EEB_INTROSPECTIVE && !is_final) {
                launch_gather_rows(cur.x, alt.x, more ? h_cur : nullptr, h_alt, (int)hrow, I.src, alt.n_active,
                                   batch, D, s);
                count(c, kCatHead, 1);
                std::swap(cur, alt);
                std::swap(h_cur, h_alt);
            }
            if (cond) s = open_cond_body(c, da.cond);
            ++hi;
        }
    }
    s = close_cond_bodies(c);  // finalize runs whatever the conditionals decided
    {
        Timer t(c, kCatOther);
        launch_finalize(batch, d.n_exits, o, I.slot, I.pos, m.kv_depth.as<uint8_t>(), d.max_seq_len,
                        policy == EEB_PROFILE ? L : 0, s);
        count(c, kCatOther, 1);
    }
}

// ---------------------------------------------------------------------------
// Prefill chunk: `rows` prompt tokens (I.tok / I.slot / I.pos) through layers
// 1..depth, no exit heads.  Same layer body as the decode step, except that
// every row's K/V is appended before the attention (rows of one sequence in
// the chunk attend to each other) and the positions are marked computed to
// `depth` up front.
// ---------------------------------------------------------------------------
constexpr int kPolicyPrefill = 100;  // graph-cache key

void enqueue_prefill(eeb_ctx* c, int mi, int depth, int rows) {
    struct InPrefill {
        eeb_ctx* c;
        explicit InPrefill(eeb_ctx* cc) : c(cc) { c->in_prefill = true; }
        ~InPrefill() { c->in_prefill = false; }
    } in_prefill_scope(c);
    Model& m = model_of(c, mi);
    const eeb_model_desc& d = m.desc;
    const int D = d.d_model;
    cudaStream_t s = c->stream;
    Ints I = ints_of(c);
    RowState cur{I.nA, I.rowA, I.slotA, I.posA, c->xA.as<float>()};
    void* h = c->hn.p;
    launch_embed(d.dtype, m.emb.p, I.tok, I.slot, I.pos, rows, D, cur, s);
    launch_mark_depth(rows, I.slot, I.pos, m.kv_depth.as<uint8_t>(), d.max_seq_len, depth, s);
    // (prefill row kernels: 4 float4 groups per thread, see norm_vec)
    launch_residual_norm(d.dtype, nullptr, 0, 0, cur.n_active, rows, cur.x, D, d.norm_eps,
                         m.layers[0]->attn_norm.as<float>(), h, nullptr, nullptr, s, nullptr, 0, 4);
    count(c, kCatOther, 3);
    for (int l = 1; l <= depth; ++l) {
        const PlaneSet dn = layer_core(c, m, l, cur, h, rows, true);
        if (l < depth && dn.px)  // the next layer's attention norm (the last layer's residual is not needed)
            launch_tp_norm(d.dtype, m.pxp, dn.planes, (int64_t)rows * D, cur.n_active, rows, cur.x, D, d.norm_eps,
                           m.layers[l]->attn_norm.as<float>(), h, nullptr, nullptr, s, 4);
        else if (l < depth)
            launch_residual_norm(d.dtype, dn.base, dn.planes, (int64_t)rows * D, cur.n_active, rows, cur.x, D,
                                 d.norm_eps, m.layers[l]->attn_norm.as<float>(), h, nullptr, nullptr, s, nullptr, 0, 4);
        count(c, kCatNorm, l < depth ? 1 : 0);
    }
}

// full: a full-size chunk of its prefill.  Only those are captured into
// graphs (a serving engine's prefills of a few admitted requests come in many
// row counts and query-block layouts; each new one would pay a capture and
// instantiation of a whole-depth graph, far more than launching it once).
void run_prefill_chunk(eeb_ctx* c, int mi, int depth, int rows, bool full) {
    const bool use_graph = c->graphs_enabled && !c->profiling && full;
    if (!use_graph) {
        enqueue_prefill(c, mi, depth, rows);
        return;
    }
    GraphKey key{mi, depth, kPolicyPrefill, rows, c->gemm_tier, (uint32_t)c->pf_cur_items};
    auto it = c->graphs.find(key);
    if (it == c->graphs.end() && c->pf_seen.insert(key).second) {
        // first sighting of this chunk layout: eager (a serving engine's
        // admissions produce many one-off query-block layouts; capturing and
        // instantiating a whole-depth graph for each cost ~0.7 s of a C3 run)
        enqueue_prefill(c, mi, depth, rows);
        return;
    }
    if (it == c->graphs.end()) {
        cudaGraph_t g;
        EEB_CUDA(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
        try {
            enqueue_prefill(c, mi, depth, rows);
        } catch (...) {
            cudaStreamEndCapture(c->stream, &g);
            throw;
        }
        EEB_CUDA(cudaStreamEndCapture(c->stream, &g));
        cudaGraphExec_t ex;
        EEB_CUDA(cudaGraphInstantiate(&ex, g, 0));
        cudaGraphDestroy(g);
        it = c->graphs.emplace(key, ex).first;
    }
    EEB_CUDA(cudaGraphLaunch(it->second, c->stream));
}

void check_step_args(eeb_ctx* c, Model& m, int depth, int policy, float th, int batch) {
    const eeb_model_desc& d = m.desc;
    if (batch <= 0 || batch > d.max_slots)
        throw Error(EEB_E_DOMAIN, "batch must be in [1, max_slots]");
    if (batch > 1024) throw Error(EEB_E_DOMAIN, "batch above 1024 rows per step");
    if (!(th >= 0.f && th <= 1.f)) throw Error(EEB_E_VALIDATION, "th must be in [0,1]");
    if (policy < EEB_FLAT || policy > EEB_PROFILE) throw Error(EEB_E_DOMAIN, "unknown token policy");
    const int need = policy == EEB_FLAT ? depth : d.num_layers;
    if (policy == EEB_FLAT && (depth <= 0 || depth > d.num_layers))
        throw Error(EEB_E_DOMAIN, "serving depth " + std::to_string(depth) + " outside [1, num_layers]");
    if (m.loaded < need)
        throw Error(EEB_E_CAPACITY, "layers up to " + std::to_string(need) + " are not resident (loaded " +
                                        std::to_string(m.loaded) + ")");
    if (d.dtype == EEB_F32 && batch > 64)
        throw Error(EEB_E_DOMAIN, "f32 parity model supports at most 64 rows per step");
    if (m.tp > 1 && (batch < tc_min_rows() || c->gemm_tier == 1 || c->retain_logits))
        throw Error(EEB_E_DOMAIN, "tensor-parallel steps need the tensor-core tier (batch >= " +
                                      std::to_string(tc_min_rows()) + ", no logit retention)");
    (void)c;
}

void run_step(eeb_ctx* c, int mi, int depth, int policy, float th, int batch) {
    Model& m = model_of(c, mi);
    if (c->stamp_cap > 0) stamp_reset(c);
    const bool use_graph = c->graphs_enabled && !c->profiling && !c->retain_logits;
    if (!use_graph) {
        c->step_launches = 0;
        StampSession ss(c);
        enqueue_step(c, mi, depth, policy, th, batch);
        if (ss.on) c->stamp_last = {ss.st.kernels, ss.st.cats};
        return;
    }
    uint32_t thb;
    std::memcpy(&thb, &th, 4);
    GraphKey key{mi, policy == EEB_FLAT ? depth : 0, policy, batch, c->gemm_tier, thb};
    auto it = c->graphs.find(key);
    if (it == c->graphs.end()) {
        c->step_launches = 0;
        cudaGraph_t g;
        EEB_CUDA(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
        c->capturing = true;
        try {
            StampSession ss(c);
            enqueue_step(c, mi, depth, policy, th, batch);
            if (ss.on) c->stamp_kernels[key] = {ss.st.kernels, ss.st.cats};
        } catch (...) {
            c->capturing = false;
            while (c->cond_open > 0) {
                --c->cond_open;
                cudaGraph_t ig;
                cudaStreamEndCapture(c->cond_streams[c->cond_open], &ig);
            }
            c->stream = c->main_stream;
            cudaStreamEndCapture(c->stream, &g);
            throw;
        }
        c->capturing = false;
        EEB_CUDA(cudaStreamEndCapture(c->stream, &g));
        cudaGraphExec_t ex;
        EEB_CUDA(cudaGraphInstantiate(&ex, g, 0));
        cudaGraphDestroy(g);
        it = c->graphs.emplace(key, ex).first;
    }
    (void)m;
    if (c->stamp_cap > 0) c->stamp_last = c->stamp_kernels[key];
    EEB_CUDA(cudaGraphLaunch(it->second, c->stream));
}

void harvest_profile(eeb_ctx* c) {
    if (!c->profiling) return;
    EEB_CUDA(cudaStreamSynchronize(c->stream));
    for (auto& [cat, ev] : c->ev_used) {
        float ms = 0.f;
        EEB_CUDA(cudaEventElapsedTime(&ms, ev.first, ev.second));
        c->cat_ms[cat] += ms;
        c->ev_pool.push_back(ev.first);
        c->ev_pool.push_back(ev.second);
    }
    c->ev_used.clear();
    c->steps_profiled += 1;
}

// KV pool ↔ kv_bytes_per_slot (memory_model.hpp:58-60).  Per layer and
// shard: [pages][hkv_l][page][hd]; unpaged = one page of max_seq_len
// positions per slot (slot == page), paged = n_pages pages on a free list.
void alloc_kv(eeb_ctx* c, Model& m, int page, int n_pages, bool paged) {
    const eeb_model_desc& d = m.desc;
    m.kv_page = page;
    m.kv_pages = n_pages;
    m.pages_per_seq = (d.max_seq_len + page - 1) / page;
    m.paged = paged;
    m.kv_shard_elems = (size_t)n_pages * m.hkv_l * page * m.head_dim;
    m.kv_layer_elems = m.kv_shard_elems * m.shards;
    m.k_cache.release();
    m.v_cache.release();
    m.k_cache.ensure(m.kv_layer_elems * d.num_layers * m.wbytes);
    m.v_cache.ensure(m.kv_layer_elems * d.num_layers * m.wbytes);
    // stream-ordered (the context stream is non-blocking: a legacy-stream
    // memset would not be ordered before the first step)
    EEB_CUDA(cudaMemsetAsync(m.k_cache.p, 0, m.k_cache.bytes, c->stream));  // finite values behind masked rows
    EEB_CUDA(cudaMemsetAsync(m.v_cache.p, 0, m.v_cache.bytes, c->stream));
    m.k_maps.clear();
    m.v_maps.clear();
    m.k_maps8.clear();
    m.v_maps8.clear();
    // (head_dim 80: rows of 160 B; the maps' second 64-dim box reads dims
    //  80..127 as out-of-bounds zeros — the prefill attention's padded tiles)
    if (d.dtype == EEB_BF16 && (m.head_dim == 64 || m.head_dim == 80 || m.head_dim == 128) && gemm_tc_available()) {
        m.k_maps.resize((size_t)d.num_layers * m.shards);
        m.v_maps.resize((size_t)d.num_layers * m.shards);
        m.k_maps8.resize((size_t)d.num_layers * m.shards);
        m.v_maps8.resize((size_t)d.num_layers * m.shards);
        for (int l = 0; l < d.num_layers; ++l)
            for (int sh = 0; sh < m.shards; ++sh) {
                const size_t off = ((size_t)l * m.kv_layer_elems + sh * m.kv_shard_elems) * 2;
                const size_t k = (size_t)l * m.shards + sh;
                make_kv_tensor_map(m.k_maps[k].data(), static_cast<char*>(m.k_cache.p) + off, m.head_dim, page,
                                   n_pages * m.hkv_l, 32);
                make_kv_tensor_map(m.v_maps[k].data(), static_cast<char*>(m.v_cache.p) + off, m.head_dim, page,
                                   n_pages * m.hkv_l, 32);
                make_kv_tensor_map(m.k_maps8[k].data(), static_cast<char*>(m.k_cache.p) + off, m.head_dim, page,
                                   n_pages * m.hkv_l, 8);
                make_kv_tensor_map(m.v_maps8[k].data(), static_cast<char*>(m.v_cache.p) + off, m.head_dim, page,
                                   n_pages * m.hkv_l, 8);
            }
    }
    m.h_table.assign((size_t)d.max_slots * m.pages_per_seq, paged ? -1 : 0);
    m.slot_npages.assign(d.max_slots, 0);
    m.free_pages.clear();
    if (!paged) {
        for (int sl = 0; sl < d.max_slots; ++sl) m.h_table[sl] = sl;
    } else {
        for (int pg = n_pages - 1; pg >= 0; --pg) m.free_pages.push_back(pg);
    }
    m.page_table.ensure(m.h_table.size() * 4);
    m.table_dirty = true;
}

// Paged pool: give `slot` pages for positions [0, n_positions) (EEB_E_CAPACITY
// when the free list runs dry, like CapacityError in apply_load,
// memory_model.hpp:86-105).
void kv_reserve(Model& m, int slot, int n_positions) {
    if (!m.paged) return;
    const int need = (n_positions + m.kv_page - 1) / m.kv_page;
    int& have = m.slot_npages[slot];
    while (have < need) {
        if (m.free_pages.empty())
            throw Error(EEB_E_CAPACITY, "KV page pool exhausted (" + std::to_string(m.kv_pages) + " pages of " +
                                            std::to_string(m.kv_page) + " positions)");
        m.h_table[(size_t)slot * m.pages_per_seq + have] = m.free_pages.back();
        m.free_pages.pop_back();
        ++have;
        m.table_dirty = true;
    }
}

void kv_release(Model& m, int slot) {
    if (!m.paged) return;
    int& have = m.slot_npages[slot];
    for (int k = have - 1; k >= 0; --k) {
        int32_t& e = m.h_table[(size_t)slot * m.pages_per_seq + k];
        m.free_pages.push_back(e);
        e = -1;
    }
    have = 0;
    m.table_dirty = true;
}

// Stream-ordered upload of the page table before work that reads it.
void kv_sync_table(eeb_ctx* c, Model& m) {
    if (!m.table_dirty) return;
    EEB_CUDA(cudaMemcpyAsync(m.page_table.p, m.h_table.data(), m.h_table.size() * 4, cudaMemcpyHostToDevice,
                             c->stream));
    m.table_dirty = false;
}

// Peer-memory tensor parallelism: the exchange-buffer layout is a function of
// the model descriptor only, so every rank computes the same offsets.
PxLayout px_layout(const Model& m) {
    const eeb_model_desc& d = m.desc;
    PxLayout L;
    auto al = [](int64_t b) { return (b + 255) / 256 * 256; };
    int64_t off = 0;
    L.arrive = off; off += al((int64_t)kPxMaxRanks * kPxMaxCtas * 4);
    L.pushed = off; off += al((int64_t)kPxMaxRanks * kPxMaxCtas * 4);
    L.epoch = off; off += al((int64_t)kPxMaxCtas * 4);
    L.g_arrive = off; off += al((int64_t)kPxMaxRanks * kPxGatherCtas * 4);
    L.g_epoch = off; off += al((int64_t)kPxGatherCtas * 4);
    L.rows = std::max(d.max_slots, kPxMaxCtas);
    L.planes_elems = (int64_t)16 * L.rows * d.d_model;
    L.planes = off; off += al(L.planes_elems * 4);
    L.red = off; off += al((int64_t)L.rows * d.d_model * 4);
    L.head_elems = (int64_t)d.max_slots * ((m.v_l + 127) / 128) * 4;
    L.head = off; off += al(L.head_elems * 4);
    L.bytes = off;
    return L;
}

}  // namespace

Stamp stamp_next(const void* kernel) {
    Stamp s;
    StampState* g = g_stamp;
    if (!g || (int)g->kernels.size() >= g->cap) return s;
    s.buf = g->buf;
    s.slot = (int)g->kernels.size();
    s.end_off = (int64_t)g->cap * kStampCtas;
    g->kernels.push_back(kernel);
    g->cats.push_back(-1);
    return s;
}

}  // namespace eeb

using namespace eeb;

extern "C" {

int eeb_abi_version(void) { return EEB_ABI_VERSION; }

const char* eeb_last_error(void) { return g_last_error.c_str(); }

eeb_status eeb_create(int device, eeb_ctx** out) {
    return guarded([&] {
        if (!out) throw Error(EEB_E_DOMAIN, "null output handle");
        *out = nullptr;
        int n = 0;
        EEB_CUDA(cudaGetDeviceCount(&n));
        if (device < 0 || device >= n) throw Error(EEB_E_DOMAIN, "no CUDA device " + std::to_string(device));
        EEB_CUDA(cudaSetDevice(device));
        cudaDeviceProp prop;
        EEB_CUDA(cudaGetDeviceProperties(&prop, device));
        if (prop.major < 10)
            throw Error(EEB_E_CUDA, std::string("eeb targets sm_100a (B200); device is ") + prop.name);
        auto c = std::make_unique<eeb_ctx>();
        c->device = device;
        c->num_sms = prop.multiProcessorCount;
        EEB_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        EEB_CUDA(cudaStreamCreateWithFlags(&c->load_stream, cudaStreamNonBlocking));
        c->main_stream = c->stream;
        // Under Nsight Compute (its injection sets NV_COMPUTE_PROFILER_PERFWORKS_DIR)
        // the step runs as plain stream launches: ncu fails to replay this
        // build's graph-captured tcgen05 GEMM node (LaunchFailed); the kernels
        // are the same either way.  eeb_set_graphs(ctx, 1) still forces graphs.
        if (std::getenv("NV_COMPUTE_PROFILER_PERFWORKS_DIR")) c->graphs_enabled = 0;
        *out = c.release();
    });
}

void eeb_destroy(eeb_ctx* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    for (auto& [k, g] : c->graphs) cudaGraphExecDestroy(g);
    for (auto ev : c->ev_pool) cudaEventDestroy(ev);
    if (c->nccl) nccl().comm_destroy(c->nccl);
    for (auto& [k, pl] : c->lt_plans) {
        if (pl.a) cublasLtMatrixLayoutDestroy(pl.a);
        if (pl.b) cublasLtMatrixLayoutDestroy(pl.b);
        if (pl.d) cublasLtMatrixLayoutDestroy(pl.d);
        if (pl.op) cublasLtMatmulDescDestroy(pl.op);
    }
    if (c->lt) cublasLtDestroy(c->lt);
    if (c->pin) cudaFreeHost(c->pin);
    if (c->pf_pin) cudaFreeHost(c->pf_pin);
    for (auto& m : c->models) {
        if (m && m->pending) {
            cudaEventSynchronize(m->pending->t1);
            eeb::settle_pending(*m);
        }
    }
    c->models.clear();
    cudaStreamDestroy(c->stream);
    cudaStreamDestroy(c->load_stream);
    for (cudaStream_t cs : c->cond_streams) cudaStreamDestroy(cs);
    delete c;
}

eeb_status eeb_model_register(eeb_ctx* c, const eeb_model_desc* desc, int* model) {
    return guarded([&] {
        if (!c || !desc || !model) throw Error(EEB_E_DOMAIN, "null argument");
        validate_desc(*desc);
        EEB_CUDA(cudaSetDevice(c->device));
        auto m = std::make_unique<Model>();
        m->desc = *desc;
        m->exits.assign(desc->exit_layers, desc->exit_layers + desc->n_exits);
        m->desc.exit_layers = m->exits.data();
        if (desc->exit_coverage) m->coverage.assign(desc->exit_coverage, desc->exit_coverage + desc->n_exits);
        else m->coverage = default_coverage(desc->n_exits);
        m->desc.exit_coverage = m->coverage.data();
        if (m->desc.norm_eps <= 0.f) m->desc.norm_eps = 1e-5f;
        if (m->desc.rope_theta <= 0.f) m->desc.rope_theta = 10000.f;
        const eeb_model_desc& d = m->desc;
        m->alphas = synth::head_alphas(d.d_model, d.vocab, d.num_layers, m->exits, m->coverage, d.design_th);
        m->head_dim = d.d_model / d.n_heads;
        m->dq = d.n_heads * m->head_dim;
        m->dkv = d.n_kv_heads * m->head_dim;
        m->up_rows = d.mlp_kind == EEB_MLP_SWIGLU ? 2 * d.d_ffn : d.d_ffn;
        m->wbytes = d.dtype == EEB_BF16 ? 2 : 4;
        m->tp = std::max(1, d.tp_size);
        m->rank = m->tp > 1 ? d.tp_rank : 0;
        m->shards = m->tp > 1 && m->rank < 0 ? m->tp : 1;
        m->hq_l = d.n_heads / m->tp;
        m->hkv_l = d.n_kv_heads / m->tp;
        m->dq_l = m->hq_l * m->head_dim;
        m->dkv_l = m->hkv_l * m->head_dim;
        m->f_l = d.d_ffn / m->tp;
        m->up_l = m->up_rows / m->tp;
        m->v_l = d.vocab / m->tp;
        if (m->head_dim % 16 != 0 || m->head_dim > 128) throw Error(EEB_E_VALIDATION, "head_dim must be a multiple of 16, <= 128");
        alloc_kv(c, *m, d.max_seq_len, d.max_slots, false);
        m->pool = &c->wpool;
        m->emb.pool = &c->wpool;
        m->kv_depth.ensure((size_t)d.max_slots * d.max_seq_len);
        EEB_CUDA(cudaMemsetAsync(m->kv_depth.p, 0, m->kv_depth.bytes, c->stream));
        EEB_CUDA(cudaStreamSynchronize(c->stream));
        // RoPE tables in f64 then rounded (restated identically by the oracle).
        const int half = m->head_dim / 2;
        std::vector<float> cs((size_t)d.max_seq_len * half), sn((size_t)d.max_seq_len * half);
        for (int p = 0; p < d.max_seq_len; ++p)
            for (int j = 0; j < half; ++j) {
                const double inv = std::pow((double)d.rope_theta, -2.0 * j / (double)m->head_dim);
                const double ang = (double)p * inv;
                cs[(size_t)p * half + j] = (float)std::cos(ang);
                sn[(size_t)p * half + j] = (float)std::sin(ang);
            }
        m->rope_cos.ensure(cs.size() * 4);
        m->rope_sin.ensure(sn.size() * 4);
        EEB_CUDA(cudaMemcpy(m->rope_cos.p, cs.data(), cs.size() * 4, cudaMemcpyHostToDevice));
        EEB_CUDA(cudaMemcpy(m->rope_sin.p, sn.data(), sn.size() * 4, cudaMemcpyHostToDevice));
        c->models.push_back(std::move(m));
        *model = (int)c->models.size() - 1;
    });
}

eeb_status eeb_load_layers(eeb_ctx* c, int model, int to_depth) {
    return guarded([&] {
        Model& m = model_of(c, model);
        EEB_CUDA(cudaSetDevice(c->device));
        drop_graphs(c, model);
        load_to(c, m, to_depth);
    });
}

eeb_status eeb_evict(eeb_ctx* c, int model) { return eeb_load_layers(c, model, 0); }

eeb_status eeb_weight_reserve(eeb_ctx* c, int model, int depth) {
    return guarded([&] {
        Model& m = model_of(c, model);
        const eeb_model_desc& d = m.desc;
        if (depth < 0 || depth > d.num_layers) throw Error(EEB_E_DOMAIN, "depth outside [0, num_layers]");
        EEB_CUDA(cudaSetDevice(c->device));
        // allocate what a load to `depth` would (beyond what is resident) and
        // hand it straight to the context's block pool
        std::vector<std::unique_ptr<LayerWeights>> tmp;
        for (int l = (int)m.layers.size() + 1; l <= depth; ++l) tmp.push_back(alloc_layer(m));
        if (m.loaded == 0 && depth > 0) {
            const int D = d.d_model;
            DevBuf e(m.pool);
            e.ensure((size_t)d.vocab * D * m.wbytes);
            std::vector<std::unique_ptr<DevBuf>> hs;
            for (int x = 0; x < d.n_exits; ++x) {
                hs.push_back(std::make_unique<DevBuf>(m.pool));
                hs.back()->ensure((size_t)m.v_l * D * m.wbytes * m.shards);
                hs.push_back(std::make_unique<DevBuf>(m.pool));
                hs.back()->ensure((size_t)D * 4);
            }
        }
    });
}

eeb_status eeb_host_stage(eeb_ctx* c, int model, int depth) {
    return guarded([&] {
        Model& m = model_of(c, model);
        EEB_CUDA(cudaSetDevice(c->device));
        host_stage(c, m, depth);
    });
}

eeb_status eeb_weight_layout(eeb_ctx* c, int model, eeb_weight_layout_t* out) {
    return guarded([&] {
        Model& m = model_of(c, model);
        if (!out) throw Error(EEB_E_DOMAIN, "null argument");
        std::vector<size_t> lo, bo;
        out->layer_bytes = (int64_t)packed_offsets(layer_part_bytes(m), &lo);
        out->base_bytes = (int64_t)packed_offsets(base_part_bytes(m), &bo);
        for (int k = 0; k < 6; ++k) out->layer_off[k] = (int64_t)lo[k];
        for (int k = 0; k < 1 + 2 * 64; ++k) out->base_off[k] = k < (int)bo.size() ? (int64_t)bo[k] : -1;
    });
}

eeb_status eeb_host_stage_layer(eeb_ctx* c, int model, int layer, const void* host, int64_t bytes) {
    return guarded([&] {
        Model& m = model_of(c, model);
        require_single_shard(m);
        if (layer < 1 || layer > m.desc.num_layers) throw Error(EEB_E_DOMAIN, "layer outside [1, num_layers]");
        if (layer > (int)m.host.layers.size() + 1)
            throw Error(EEB_E_DOMAIN, "host tier is a prefix: stage layer " + std::to_string(m.host.layers.size() + 1) +
                                          " first");
        EEB_CUDA(cudaSetDevice(c->device));
        settle_pending(m);
        auto b = blob_from_host(layer_part_bytes(m), host, bytes);
        if (layer == (int)m.host.layers.size() + 1) m.host.layers.push_back(std::move(b));
        else m.host.layers[layer - 1] = std::move(b);
        if (layer <= (int)m.layers.size()) {  // resident: refresh the device copy
            EEB_CUDA(cudaStreamSynchronize(c->stream));
            m.layers[layer - 1] = layer_from_host(m, layer, c->stream);
            EEB_CUDA(cudaStreamSynchronize(c->stream));
            drop_graphs(c, model);
        }
    });
}

eeb_status eeb_host_stage_base(eeb_ctx* c, int model, const void* host, int64_t bytes) {
    return guarded([&] {
        Model& m = model_of(c, model);
        require_single_shard(m);
        EEB_CUDA(cudaSetDevice(c->device));
        settle_pending(m);
        m.host.base = blob_from_host(base_part_bytes(m), host, bytes);
        if (m.loaded > 0) {  // resident: refresh the device copy
            EEB_CUDA(cudaStreamSynchronize(c->stream));
            base_from_host(m, c->stream);
            EEB_CUDA(cudaStreamSynchronize(c->stream));
            drop_graphs(c, model);
        }
    });
}

eeb_status eeb_load_layers_from(eeb_ctx* c, int model, int from, int to, const void* host, int64_t bytes) {
    return guarded([&] {
        Model& m = model_of(c, model);
        require_single_shard(m);
        if (from < 1 || to < from || to > m.desc.num_layers) throw Error(EEB_E_DOMAIN, "need 1 <= from <= to <= num_layers");
        if (from > (int)m.host.layers.size() + 1 || from > m.loaded + 1)
            throw Error(EEB_E_DOMAIN, "layers are loaded as a prefix: from must be <= loaded_depth + 1");
        const int64_t per = (int64_t)packed_offsets(layer_part_bytes(m), nullptr);
        if (!host || bytes != per * (to - from + 1))
            throw Error(EEB_E_VALIDATION, "buffer must hold " + std::to_string(to - from + 1) + " packed layers of " +
                                              std::to_string(per) + " bytes");
        EEB_CUDA(cudaSetDevice(c->device));
        settle_pending(m);
        for (int l = from; l <= to; ++l) {
            auto b = blob_from_host(layer_part_bytes(m), static_cast<const char*>(host) + (l - from) * per, per);
            if (l == (int)m.host.layers.size() + 1) m.host.layers.push_back(std::move(b));
            else m.host.layers[l - 1] = std::move(b);
        }
        drop_graphs(c, model);
        while ((int)m.layers.size() >= from) m.layers.pop_back();  // reloaded from the new host copies
        m.loaded = (int)m.layers.size();
        load_to(c, m, std::max(to, m.loaded));
    });
}

eeb_status eeb_load_layers_async(eeb_ctx* c, int model, int to_depth) {
    return guarded([&] {
        Model& m = model_of(c, model);
        EEB_CUDA(cudaSetDevice(c->device));
        drop_graphs(c, model);
        load_async(c, m, to_depth);
    });
}

eeb_status eeb_load_wait(eeb_ctx* c, int model, double* seconds, int64_t* bytes) {
    return guarded([&] {
        Model& m = model_of(c, model);
        EEB_CUDA(cudaSetDevice(c->device));
        settle_pending(m);
        if (seconds) *seconds = m.last_load_s;
        if (bytes) *bytes = m.last_load_bytes;
    });
}

eeb_status eeb_loaded_depth(eeb_ctx* c, int model, int* depth) {
    return guarded([&] {
        if (!depth) throw Error(EEB_E_DOMAIN, "null output");
        *depth = model_of(c, model).loaded;
    });
}

eeb_status eeb_weight_bytes(eeb_ctx* c, int model, int depth, int64_t* bytes) {
    return guarded([&] {
        Model& m = model_of(c, model);
        if (!bytes) throw Error(EEB_E_DOMAIN, "null output");
        if (depth < 0 || depth > m.desc.num_layers) throw Error(EEB_E_DOMAIN, "depth outside [0, num_layers]");
        *bytes = weight_bytes_at(m, depth);
    });
}

eeb_status eeb_reset_slots(eeb_ctx* c, int model, int32_t n, const int32_t* slot_ids) {
    return guarded([&] {
        Model& m = model_of(c, model);
        for (int i = 0; i < n; ++i) {
            if (slot_ids[i] < 0 || slot_ids[i] >= m.desc.max_slots) throw Error(EEB_E_DOMAIN, "slot out of range");
            EEB_CUDA(cudaMemsetAsync(m.kv_depth.as<uint8_t>() + (size_t)slot_ids[i] * m.desc.max_seq_len, 0,
                                     m.desc.max_seq_len, c->stream));
        }
        EEB_CUDA(cudaStreamSynchronize(c->stream));
    });
}

static void validate_rows_host(const Model& m, int batch, const int32_t* slot, const int32_t* tok,
                               const int32_t* pos) {
    thread_local std::vector<uint8_t> seen;
    seen.assign((size_t)m.desc.max_slots, 0);
    for (int i = 0; i < batch; ++i) {
        if (slot[i] < 0 || slot[i] >= m.desc.max_slots) throw Error(EEB_E_DOMAIN, "slot id out of range");
        if (tok[i] < 0 || tok[i] >= m.desc.vocab) throw Error(EEB_E_DOMAIN, "token id out of range");
        if (pos[i] < 0 || pos[i] >= m.desc.max_seq_len) throw Error(EEB_E_DOMAIN, "position out of range");
        if (seen[slot[i]]++) throw Error(EEB_E_VALIDATION, "duplicate slot id in one step");
    }
}

eeb_status eeb_decode_step(eeb_ctx* c, int model, int depth, int policy, float th, int32_t batch,
                           const int32_t* slot_ids, const int32_t* input_tokens, const int32_t* positions,
                           eeb_step_out* out) {
    return guarded([&] {
        Model& m = model_of(c, model);
        if (!slot_ids || !input_tokens || !positions) throw Error(EEB_E_DOMAIN, "null input array");
        check_step_args(c, m, depth, policy, th, batch);
        validate_rows_host(m, batch, slot_ids, input_tokens, positions);
        for (int i = 0; i < batch; ++i) kv_reserve(m, slot_ids[i], positions[i] + 1);
        kv_sync_table(c, m);
        EEB_CUDA(cudaSetDevice(c->device));
        ensure_workspace(c, m, batch);
        wait_layers(c, m, policy == EEB_FLAT ? depth : m.desc.num_layers);
        Ints I = ints_of(c);
        cudaStream_t s = c->stream;
        // inputs: pinned staging → device
        // inputs: the three row arrays are adjacent on the device (stride
        // cap_rows): staged the same way in pinned memory, one H2D copy
        const int R = c->cap_rows;
        char* pin = static_cast<char*>(c->pin);
        int32_t* pin_in = reinterpret_cast<int32_t*>(pin);
        std::memcpy(pin_in, input_tokens, (size_t)batch * 4);
        std::memcpy(pin_in + R, slot_ids, (size_t)batch * 4);
        std::memcpy(pin_in + 2 * R, positions, (size_t)batch * 4);
        EEB_CUDA(cudaMemcpyAsync(I.tok, pin_in, (size_t)(2 * R + batch) * 4, cudaMemcpyHostToDevice, s));
        run_step(c, model, depth, policy, th, batch);
        // outputs: one D2H copy of the output block into pinned staging, then
        // the requested arrays to the caller
        const OutLayout L(R, 64);
        char* po = reinterpret_cast<char*>(((uintptr_t)(pin + (size_t)R * 12) + 255) & ~(uintptr_t)255);
        const int ne = m.desc.n_exits;
        if (out) {
            const size_t n = policy == EEB_PROFILE ? L.total : L.common_end;
            EEB_CUDA(cudaMemcpyAsync(po, c->o_all.p, n, cudaMemcpyDeviceToHost, s));
        }
        EEB_CUDA(cudaStreamSynchronize(s));
        if (out) {
            auto put = [&](void* dst, size_t off, size_t bytes) {
                if (dst) std::memcpy(dst, po + off, bytes);
            };
            put(out->exit_layer, L.exit, (size_t)batch * 4);
            put(out->token_id, L.tok, (size_t)batch * 4);
            put(out->confidence, L.conf, (size_t)batch * 4);
            put(out->logprob, L.logp, (size_t)batch * 4);
            put(out->breached, L.breach, (size_t)batch);
            put(out->unchanged, L.unch, (size_t)batch);
            put(out->hist, L.hist, (size_t)ne * 8);
            put(out->n_breached, L.nbr, 8);
            put(out->sum_logprob, L.sum, 8);
            if (policy == EEB_PROFILE) {
                put(out->head_token, L.htok, (size_t)batch * ne * 4);
                put(out->head_confidence, L.hconf, (size_t)batch * ne * 4);
                put(out->head_logprob, L.hlogp, (size_t)batch * ne * 4);
            }
        }
        harvest_profile(c);
    });
}

eeb_status eeb_decode_step_device(eeb_ctx* c, int model, int depth, int policy, float th, int32_t batch,
                                  const int32_t* d_slot, const int32_t* d_tok, const int32_t* d_pos,
                                  eeb_step_out* d_out) {
    return guarded([&] {
        Model& m = model_of(c, model);
        if (!d_slot || !d_tok || !d_pos) throw Error(EEB_E_DOMAIN, "null input array");
        check_step_args(c, m, depth, policy, th, batch);
        EEB_CUDA(cudaSetDevice(c->device));
        ensure_workspace(c, m, batch);
        wait_layers(c, m, policy == EEB_FLAT ? depth : m.desc.num_layers);
        kv_sync_table(c, m);  // pages reserved with eeb_kv_reserve (positions are device-side here)
        Ints I = ints_of(c);
        cudaStream_t s = c->stream;
        EEB_CUDA(cudaMemcpyAsync(I.tok, d_tok, (size_t)batch * 4, cudaMemcpyDeviceToDevice, s));
        EEB_CUDA(cudaMemcpyAsync(I.slot, d_slot, (size_t)batch * 4, cudaMemcpyDeviceToDevice, s));
        EEB_CUDA(cudaMemcpyAsync(I.pos, d_pos, (size_t)batch * 4, cudaMemcpyDeviceToDevice, s));
        run_step(c, model, depth, policy, th, batch);
        if (d_out) {
            const int ne = m.desc.n_exits;
            const StepOutDev od = out_dev(c);
            auto cp = [&](void* dst, const void* src, size_t bytes) {
                if (dst) EEB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, s));
            };
            cp(d_out->exit_layer, od.exit_layer, (size_t)batch * 4);
            cp(d_out->token_id, od.token_id, (size_t)batch * 4);
            cp(d_out->confidence, od.confidence, (size_t)batch * 4);
            cp(d_out->logprob, od.logprob, (size_t)batch * 4);
            cp(d_out->breached, od.breached, (size_t)batch);
            cp(d_out->unchanged, od.unchanged, (size_t)batch);
            cp(d_out->hist, od.hist, (size_t)ne * 8);
            cp(d_out->n_breached, od.n_breached, 8);
            cp(d_out->sum_logprob, od.sum_logprob, 8);
            if (policy == EEB_PROFILE) {
                cp(d_out->head_token, od.head_token, (size_t)batch * ne * 4);
                cp(d_out->head_confidence, od.head_confidence, (size_t)batch * ne * 4);
                cp(d_out->head_logprob, od.head_logprob, (size_t)batch * ne * 4);
            }
        }
        if (c->profiling) harvest_profile(c);
    });
}

eeb_status eeb_prefill(eeb_ctx* c, int model, int depth, int32_t n_seq, const int32_t* slot_ids,
                       const int32_t* start_pos, const int32_t* lens, const int32_t* tokens) {
    return guarded([&] {
        Model& m = model_of(c, model);
        const eeb_model_desc& d = m.desc;
        if (n_seq <= 0) throw Error(EEB_E_DOMAIN, "n_seq must be positive");
        if (!slot_ids || !start_pos || !lens || !tokens) throw Error(EEB_E_DOMAIN, "null input array");
        if (depth <= 0 || depth > d.num_layers)
            throw Error(EEB_E_DOMAIN, "prefill depth " + std::to_string(depth) + " outside [1, num_layers]");
        if (m.loaded < depth)
            throw Error(EEB_E_CAPACITY, "layers up to " + std::to_string(depth) + " are not resident (loaded " +
                                            std::to_string(m.loaded) + ")");
        int64_t total = 0;
        for (int k = 0; k < n_seq; ++k) {
            if (slot_ids[k] < 0 || slot_ids[k] >= d.max_slots) throw Error(EEB_E_DOMAIN, "slot id out of range");
            if (lens[k] < 0 || start_pos[k] < 0 || (int64_t)start_pos[k] + lens[k] > d.max_seq_len)
                throw Error(EEB_E_DOMAIN, "prompt exceeds max_seq_len");
            for (int j = 0; j < k; ++j)
                if (slot_ids[j] == slot_ids[k]) throw Error(EEB_E_VALIDATION, "duplicate slot id in one prefill");
            total += lens[k];
        }
        for (int64_t t = 0; t < total; ++t)
            if (tokens[t] < 0 || tokens[t] >= d.vocab) throw Error(EEB_E_DOMAIN, "token id out of range");
        if (total == 0) return;
        for (int k = 0; k < n_seq; ++k) kv_reserve(m, slot_ids[k], start_pos[k] + lens[k]);
        kv_sync_table(c, m);
        EEB_CUDA(cudaSetDevice(c->device));
        wait_layers(c, m, depth);
        static const int env_chunk = std::getenv("EEB_PREFILL_CHUNK") ? std::atoi(std::getenv("EEB_PREFILL_CHUNK")) : 0;
        // bf16: 1024-row chunks when the layer GEMMs run on cuBLASLt (fewer
        // re-streams of the weights), else 256 (tcgen05 N <= 256); f32: the
        // CUDA-core tier serves <= 64 rows per pass
        const bool lt = d.dtype == EEB_BF16 && c->gemm_tier != 1 && prefill_lt_ready(c);
        const int lt_max = m.tp > 1 ? 1024 : 4096;  // (TP exchange: one CTA per row, <= 1024)
        const int chunk = d.dtype == EEB_BF16 ? (env_chunk >= 16 && env_chunk <= (lt ? lt_max : 256) ? env_chunk
                                                                                                     : (lt ? 1024 : 256))
                                              : 128;
        ensure_workspace(c, m, (int)std::min<int64_t>(chunk, total));
        // (tok, slot, pos) of every prompt token: one pinned staging + one H2D,
        // then a device-to-device slice per chunk.
        // query blocks of every chunk for the tensor-core prefill attention:
        // runs of consecutive rows of one sequence (consecutive positions),
        // at most 64 rows, never across a chunk boundary
        std::vector<std::vector<int4>> chunk_items;
        {
            int64_t t0 = 0;
            for (int k = 0; k < n_seq; t0 += lens[k], ++k)
                for (int j = 0; j < lens[k];) {
                    const int64_t row = t0 + j;
                    const int64_t ci = row / chunk;
                    while ((int64_t)chunk_items.size() <= ci) chunk_items.emplace_back();
                    const int in_chunk = (int)(row - ci * chunk);
                    const int n = (int)std::min<int64_t>({64, lens[k] - j, (ci + 1) * chunk - row});
                    chunk_items[ci].push_back(make_int4(in_chunk, n, slot_ids[k], start_pos[k] + j));
                    j += n;
                }
        }
        size_t max_items = 0;
        for (const auto& v : chunk_items) max_items = std::max(max_items, v.size());
        const size_t item_bytes = chunk_items.size() * (max_items + 1) * sizeof(int4);
        const size_t meta = (size_t)total * 3 * 4;
        const size_t meta_al = ((meta + 15) / 16) * 16;
        if (meta_al + item_bytes > c->pf_pin_bytes) {
            if (c->pf_pin) cudaFreeHost(c->pf_pin);
            c->pf_pin = nullptr;
            EEB_CUDA(cudaMallocHost(&c->pf_pin, meta_al + item_bytes));
            c->pf_pin_bytes = meta_al + item_bytes;
        }
        int32_t* ht = static_cast<int32_t*>(c->pf_pin);
        int32_t* hs = ht + total;
        int32_t* hp = hs + total;
        int64_t t = 0;
        for (int k = 0; k < n_seq; ++k)
            for (int j = 0; j < lens[k]; ++j, ++t) {
                ht[t] = tokens[t];
                hs[t] = slot_ids[k];
                hp[t] = start_pos[k] + j;
            }
        // per chunk: max_items + 1 int4 (the blocks, then their count in .x)
        int4* hi = reinterpret_cast<int4*>(static_cast<char*>(c->pf_pin) + meta_al);
        for (size_t ci = 0; ci < chunk_items.size(); ++ci) {
            int4* dst = hi + ci * (max_items + 1);
            for (size_t q = 0; q < chunk_items[ci].size(); ++q) dst[q] = chunk_items[ci][q];
            dst[chunk_items[ci].size()] = make_int4((int)chunk_items[ci].size(), 0, 0, 0);
        }
        c->pf_meta.ensure(meta_al + item_bytes);
        int32_t* dm = c->pf_meta.as<int32_t>();
        cudaStream_t s = c->stream;
        EEB_CUDA(cudaMemcpyAsync(dm, ht, meta_al + item_bytes, cudaMemcpyHostToDevice, s));
        const int4* di = reinterpret_cast<const int4*>(reinterpret_cast<const char*>(dm) + meta_al);
        c->pf_items.ensure((max_items + 1) * sizeof(int4));
        Ints I = ints_of(c);
        for (int64_t c0 = 0; c0 < total; c0 += chunk) {
            const int rows = (int)std::min<int64_t>(chunk, total - c0);
            const size_t ci = (size_t)(c0 / chunk);
            EEB_CUDA(cudaMemcpyAsync(I.tok, dm + c0, (size_t)rows * 4, cudaMemcpyDeviceToDevice, s));
            EEB_CUDA(cudaMemcpyAsync(I.slot, dm + total + c0, (size_t)rows * 4, cudaMemcpyDeviceToDevice, s));
            EEB_CUDA(cudaMemcpyAsync(I.pos, dm + 2 * total + c0, (size_t)rows * 4, cudaMemcpyDeviceToDevice, s));
            // this chunk's blocks, then the count right after them (the kernel's pf_n_items)
            const int n_items = (int)chunk_items[ci].size();
            EEB_CUDA(cudaMemcpyAsync(c->pf_items.p, di + ci * (max_items + 1), (size_t)n_items * sizeof(int4),
                                     cudaMemcpyDeviceToDevice, s));
            EEB_CUDA(cudaMemcpyAsync(c->pf_items.as<int4>() + n_items, di + ci * (max_items + 1) + n_items,
                                     sizeof(int4), cudaMemcpyDeviceToDevice, s));
            c->pf_cur_items = n_items;
            run_prefill_chunk(c, model, depth, rows, rows == chunk);
        }
        c->pf_cur_items = 0;
        EEB_CUDA(cudaStreamSynchronize(s));
    });
}

eeb_status eeb_synchronize(eeb_ctx* c) {
    return guarded([&] {
        if (!c) throw Error(EEB_E_DOMAIN, "null context");
        EEB_CUDA(cudaStreamSynchronize(c->stream));
    });
}

eeb_status eeb_set_graphs(eeb_ctx* c, int enable) {
    return guarded([&] {
        if (!c) throw Error(EEB_E_DOMAIN, "null context");
        c->graphs_enabled = enable ? 1 : 0;
    });
}

eeb_status eeb_debug_stamps(eeb_ctx* c, int max_launches) {
    return guarded([&] {
        if (!c || max_launches < 0 || max_launches > 4096) throw Error(EEB_E_DOMAIN, "bad argument");
        EEB_CUDA(cudaSetDevice(c->device));
        EEB_CUDA(cudaStreamSynchronize(c->stream));
        drop_graphs(c);  // stamped and plain graphs differ in their kernel arguments
        c->stamp_kernels.clear();
        c->stamp_last = {};
        c->stamp_cap = max_launches;
        if (max_launches > 0) {
            c->stamp_buf.release();
            c->stamp_buf.ensure((size_t)max_launches * kStampCtas * 4 * 8);
        } else {
            c->stamp_buf.release();
        }
    });
}

eeb_status eeb_debug_stamps_read(eeb_ctx* c, char* json_out, int64_t cap) {
    return guarded([&] {
        if (!c || !json_out) throw Error(EEB_E_DOMAIN, "null argument");
        if (c->stamp_cap <= 0) throw Error(EEB_E_DOMAIN, "stamping is off (eeb_debug_stamps)");
        EEB_CUDA(cudaStreamSynchronize(c->stream));
        const size_t cells = (size_t)c->stamp_cap * kStampCtas;
        std::vector<unsigned long long> h(4 * cells);
        EEB_CUDA(cudaMemcpy(h.data(), c->stamp_buf.p, h.size() * 8, cudaMemcpyDeviceToHost));
        std::string j = "{\"launches\": [";
        unsigned long long t0 = ~0ull;
        for (size_t i = 0; i < c->stamp_last.first.size(); ++i)
            for (int k = 0; k < kStampCtas; ++k) t0 = std::min(t0, h[i * kStampCtas + k]);
        for (size_t i = 0; i < c->stamp_last.first.size(); ++i) {
            unsigned long long st = ~0ull, en = 0, wt = ~0ull, mk = 0;
            int ctas = 0;
            for (int k = 0; k < kStampCtas; ++k) {
                const unsigned long long a = h[i * kStampCtas + k], b = h[cells + i * kStampCtas + k];
                wt = std::min(wt, h[2 * cells + i * kStampCtas + k]);
                mk = std::max(mk, h[3 * cells + i * kStampCtas + k]);
                if (a != ~0ull) {
                    ++ctas;
                    st = std::min(st, a);
                }
                en = std::max(en, b);
            }
            const char* name = nullptr;
            if (cudaFuncGetName(&name, c->stamp_last.first[i]) != cudaSuccess || !name) name = "?";
            const int cat = c->stamp_last.second[i];
            char buf[512];
            std::snprintf(buf, sizeof buf,
                          "%s{\"kernel\": \"%s\", \"cat\": \"%s\", \"start_ns\": %lld, \"end_ns\": %lld, "
                          "\"wait_ns\": %lld, \"mark_ns\": %lld, \"ctas\": %d}",
                          i ? ", " : "", name, cat >= 0 ? kCatNames[cat] : "?", ctas ? (long long)(st - t0) : -1LL,
                          ctas ? (long long)(en - t0) : -1LL, wt != ~0ull ? (long long)(wt - t0) : -1LL,
                          mk ? (long long)(mk - t0) : -1LL, ctas);
            j += buf;
        }
        j += "]}";
        if ((int64_t)j.size() + 1 > cap) throw Error(EEB_E_DOMAIN, "buffer too small");
        std::memcpy(json_out, j.c_str(), j.size() + 1);
    });
}

eeb_status eeb_debug_stamps_cta(eeb_ctx* c, int launch, int64_t* start_ns, int64_t* end_ns, int64_t* wait_ns,
                                int64_t* mark_ns, int n) {
    return guarded([&] {
        if (!c || c->stamp_cap <= 0) throw Error(EEB_E_DOMAIN, "stamping is off (eeb_debug_stamps)");
        if (launch < 0 || launch >= (int)c->stamp_last.first.size() || n < 0 || n > kStampCtas)
            throw Error(EEB_E_DOMAIN, "bad argument");
        EEB_CUDA(cudaStreamSynchronize(c->stream));
        const size_t cells = (size_t)c->stamp_cap * kStampCtas;
        std::vector<unsigned long long> all(cells);
        EEB_CUDA(cudaMemcpy(all.data(), c->stamp_buf.p, cells * 8, cudaMemcpyDeviceToHost));
        unsigned long long t0 = ~0ull;
        for (size_t i = 0; i < c->stamp_last.first.size() * kStampCtas; ++i) t0 = std::min(t0, all[i]);
        std::vector<unsigned long long> h(4 * (size_t)n);
        for (int w = 0; w < 4; ++w)
            EEB_CUDA(cudaMemcpy(h.data() + (size_t)w * n, c->stamp_buf.as<unsigned long long>() + w * cells +
                                (size_t)launch * kStampCtas, (size_t)n * 8, cudaMemcpyDeviceToHost));
        auto rel = [&](unsigned long long v, bool is_end) -> int64_t {
            if ((!is_end && v == ~0ull) || (is_end && v == 0)) return -1;
            return (int64_t)(v - t0);
        };
        for (int k = 0; k < n; ++k) {
            if (start_ns) start_ns[k] = rel(h[k], false);
            if (end_ns) end_ns[k] = rel(h[(size_t)n + k], true);
            if (wait_ns) wait_ns[k] = rel(h[2 * (size_t)n + k], false);
            if (mark_ns) mark_ns[k] = rel(h[3 * (size_t)n + k], true);
        }
    });
}

eeb_status eeb_set_gemm_tier(eeb_ctx* c, int tier) {
    return guarded([&] {
        if (!c) throw Error(EEB_E_DOMAIN, "null context");
        if (tier < 0 || tier > 2) throw Error(EEB_E_DOMAIN, "tier must be 0, 1 or 2");
        c->gemm_tier = tier;
    });
}

eeb_status eeb_debug_retain_logits(eeb_ctx* c, int enable) {
    return guarded([&] {
        if (!c) throw Error(EEB_E_DOMAIN, "null context");
        c->retain_logits = enable ? 1 : 0;
        drop_graphs(c);
    });
}

eeb_status eeb_debug_last_logits(eeb_ctx* c, int head, float* host_out, int64_t n) {
    return guarded([&] {
        if (!c || !host_out) throw Error(EEB_E_DOMAIN, "null argument");
        if (head < 0 || head >= (int)c->logits_keep.size() || !c->logits_keep[head]->p)
            throw Error(EEB_E_STALE, "no logits retained for that head");
        if ((size_t)n * 4 > c->logits_keep[head]->bytes) throw Error(EEB_E_DOMAIN, "n too large");
        EEB_CUDA(cudaStreamSynchronize(c->stream));
        EEB_CUDA(cudaMemcpy(host_out, c->logits_keep[head]->p, (size_t)n * 4, cudaMemcpyDeviceToHost));
    });
}

eeb_status eeb_debug_read_weight(eeb_ctx* c, int model, int tensor, int layer, int64_t offset, int64_t n,
                                 float* host_out) {
    return guarded([&] {
        Model& m = model_of(c, model);
        const void* src = nullptr;
        size_t esz = m.wbytes;
        size_t total = 0;
        if (tensor >= 100) {  // base: 100 = embedding, 200+e = head e, 300+e = head norm e
            if (m.loaded == 0) throw Error(EEB_E_STALE, "model not loaded");
            if (tensor == 100) { src = m.emb.p; total = m.emb.bytes; }
            else if (tensor >= 300) { src = m.head_norm.at(tensor - 300)->p; esz = 4; total = m.head_norm.at(tensor - 300)->bytes; }
            else { src = m.head.at(tensor - 200)->p; total = m.head.at(tensor - 200)->bytes; }
        } else {
            if (layer < 1 || layer > m.loaded) throw Error(EEB_E_STALE, "layer not resident");
            const LayerWeights& W = *m.layers[layer - 1];
            const DevBuf* b = nullptr;
            switch (tensor) {
                case synth::kAttnNorm: b = &W.attn_norm; esz = 4; break;
                case synth::kMlpNorm: b = &W.mlp_norm; esz = 4; break;
                case synth::kWqkv: b = &W.wqkv; break;
                case synth::kWo: b = &W.wo; break;
                case synth::kWup: b = &W.wup; break;
                case synth::kWdown: b = &W.wdown; break;
                default: throw Error(EEB_E_DOMAIN, "unknown tensor");
            }
            src = b->p;
            total = b->bytes;
        }
        if (offset < 0 || n < 0 || (size_t)(offset + n) * esz > total) throw Error(EEB_E_DOMAIN, "range outside tensor");
        std::vector<char> tmp((size_t)n * esz);
        EEB_CUDA(cudaStreamSynchronize(c->stream));
        EEB_CUDA(cudaMemcpy(tmp.data(), static_cast<const char*>(src) + (size_t)offset * esz, tmp.size(),
                            cudaMemcpyDeviceToHost));
        for (int64_t i = 0; i < n; ++i) {
            if (esz == 4) std::memcpy(&host_out[i], &tmp[(size_t)i * 4], 4);
            else {
                uint16_t h;
                std::memcpy(&h, &tmp[(size_t)i * 2], 2);
                uint32_t u = (uint32_t)h << 16;
                std::memcpy(&host_out[i], &u, 4);
            }
        }
    });
}

/* Paged KV pool. */
eeb_status eeb_kv_configure_pages(eeb_ctx* c, int model, int32_t page_size, int32_t n_pages) {
    return guarded([&] {
        Model& m = model_of(c, model);
        const eeb_model_desc& d = m.desc;
        if (page_size <= 0 || page_size % 64 != 0)
            throw Error(EEB_E_VALIDATION, "page_size must be a positive multiple of 64 positions");
        if (n_pages <= 0) throw Error(EEB_E_VALIDATION, "n_pages must be positive");
        if ((d.max_seq_len + page_size - 1) / page_size > 64)
            throw Error(EEB_E_VALIDATION, "at most 64 pages per sequence (max_seq_len / page_size)");
        if (d.dtype != EEB_BF16 || (m.head_dim != 64 && m.head_dim != 80 && m.head_dim != 128) ||
            !gemm_tc_available())
            throw Error(EEB_E_DOMAIN, "the paged KV pool needs a bf16 model with head_dim 64, 80 or 128");
        EEB_CUDA(cudaSetDevice(c->device));
        EEB_CUDA(cudaStreamSynchronize(c->stream));
        drop_graphs(c, model);  // captured steps hold the old KV maps and the unpaged kernel
        alloc_kv(c, m, page_size, n_pages, true);
        EEB_CUDA(cudaMemsetAsync(m.kv_depth.p, 0, m.kv_depth.bytes, c->stream));
        kv_sync_table(c, m);
        EEB_CUDA(cudaStreamSynchronize(c->stream));
    });
}

eeb_status eeb_kv_reserve(eeb_ctx* c, int model, int32_t slot, int32_t n_positions) {
    return guarded([&] {
        Model& m = model_of(c, model);
        if (slot < 0 || slot >= m.desc.max_slots) throw Error(EEB_E_DOMAIN, "slot out of range");
        if (n_positions < 0 || n_positions > m.desc.max_seq_len) throw Error(EEB_E_DOMAIN, "positions out of range");
        kv_reserve(m, slot, n_positions);
    });
}

eeb_status eeb_kv_release(eeb_ctx* c, int model, int32_t slot) {
    return guarded([&] {
        Model& m = model_of(c, model);
        if (slot < 0 || slot >= m.desc.max_slots) throw Error(EEB_E_DOMAIN, "slot out of range");
        // the released pages may be handed out by the next reservation: work
        // already queued on the context stream reads them first (stream order)
        kv_release(m, slot);
        EEB_CUDA(cudaMemsetAsync(m.kv_depth.as<uint8_t>() + (size_t)slot * m.desc.max_seq_len, 0,
                                 m.desc.max_seq_len, c->stream));
    });
}

eeb_status eeb_kv_pages(eeb_ctx* c, int model, int32_t* page_size, int32_t* n_pages, int32_t* n_free) {
    return guarded([&] {
        Model& m = model_of(c, model);
        if (page_size) *page_size = m.kv_page;
        if (n_pages) *n_pages = m.kv_pages;
        if (n_free) *n_free = m.paged ? (int32_t)m.free_pages.size() : 0;
    });
}

eeb_status eeb_debug_read_kv_span(eeb_ctx* c, int model, int layer, int slot, int pos0, int n_pos, float* host_k,
                                  float* host_v) {
    return guarded([&] {
        Model& m = model_of(c, model);
        const eeb_model_desc& d = m.desc;
        if (layer < 1 || layer > d.num_layers || slot < 0 || slot >= d.max_slots || pos0 < 0 || n_pos < 0 ||
            pos0 + n_pos > d.max_seq_len)
            throw Error(EEB_E_DOMAIN, "kv coordinate out of range");
        EEB_CUDA(cudaStreamSynchronize(c->stream));
        const int hd = m.head_dim, heads = m.shards * m.hkv_l, row = heads * hd;
        std::vector<char> tmp((size_t)m.kv_page * hd * m.wbytes);
        for (int g = 0; g < heads; ++g) {
            const int sh = g / m.hkv_l, lg = g % m.hkv_l;
            for (int p = pos0; p < pos0 + n_pos;) {  // one copy per run of positions inside a page
                const int in_page = p % m.kv_page, run = std::min(m.kv_page - in_page, pos0 + n_pos - p);
                const int32_t pg = m.h_table[(size_t)slot * m.pages_per_seq + p / m.kv_page];
                if (pg < 0) throw Error(EEB_E_DOMAIN, "kv position has no page (paged pool)");
                const size_t off = (size_t)(layer - 1) * m.kv_layer_elems + (size_t)sh * m.kv_shard_elems +
                                   (((size_t)pg * m.hkv_l + lg) * m.kv_page + in_page) * hd;
                for (int which = 0; which < 2; ++which) {
                    float* dst = which == 0 ? host_k : host_v;
                    if (!dst) continue;
                    const DevBuf& b = which == 0 ? m.k_cache : m.v_cache;
                    EEB_CUDA(cudaMemcpy(tmp.data(), static_cast<const char*>(b.p) + off * m.wbytes,
                                        (size_t)run * hd * m.wbytes, cudaMemcpyDeviceToHost));
                    for (int q = 0; q < run; ++q)
                        for (int j = 0; j < hd; ++j) {
                            float* o = &dst[(size_t)(p - pos0 + q) * row + (size_t)g * hd + j];
                            const size_t e = (size_t)q * hd + j;
                            if (m.wbytes == 4) {
                                std::memcpy(o, &tmp[e * 4], 4);
                            } else {
                                uint16_t h;
                                std::memcpy(&h, &tmp[e * 2], 2);
                                const uint32_t u = (uint32_t)h << 16;
                                std::memcpy(o, &u, 4);
                            }
                        }
                }
                p += run;
            }
        }
    });
}

eeb_status eeb_debug_read_kv(eeb_ctx* c, int model, int layer, int slot, int pos, float* host_k, float* host_v) {
    return guarded([&] {
        Model& m = model_of(c, model);
        const eeb_model_desc& d = m.desc;
        if (layer < 1 || layer > d.num_layers || slot < 0 || slot >= d.max_slots || pos < 0 || pos >= d.max_seq_len)
            throw Error(EEB_E_DOMAIN, "kv coordinate out of range");
        EEB_CUDA(cudaStreamSynchronize(c->stream));
        const int hd = m.head_dim;
        std::vector<char> tmp((size_t)hd * m.wbytes);
        // heads held here: all of them (one shard or all shards), or the
        // rank's hkv_l heads in a tensor-parallel rank context
        const int heads = m.shards * m.hkv_l;
        for (int g = 0; g < heads; ++g) {
            const int sh = g / m.hkv_l, lg = g % m.hkv_l;
            const int32_t pg = m.h_table[(size_t)slot * m.pages_per_seq + pos / m.kv_page];
            if (pg < 0) throw Error(EEB_E_DOMAIN, "kv position has no page (paged pool)");
            const size_t off = (size_t)(layer - 1) * m.kv_layer_elems + (size_t)sh * m.kv_shard_elems +
                               (((size_t)pg * m.hkv_l + lg) * m.kv_page + pos % m.kv_page) * hd;
            for (int which = 0; which < 2; ++which) {
                const DevBuf& b = which == 0 ? m.k_cache : m.v_cache;
                float* dst = (which == 0 ? host_k : host_v) + (size_t)g * hd;
                if (!dst) continue;
                EEB_CUDA(cudaMemcpy(tmp.data(), static_cast<const char*>(b.p) + off * m.wbytes, tmp.size(),
                                    cudaMemcpyDeviceToHost));
                for (int j = 0; j < hd; ++j) {
                    if (m.wbytes == 4) std::memcpy(&dst[j], &tmp[(size_t)j * 4], 4);
                    else {
                        uint16_t h;
                        std::memcpy(&h, &tmp[(size_t)j * 2], 2);
                        uint32_t u = (uint32_t)h << 16;
                        std::memcpy(&dst[j], &u, 4);
                    }
                }
            }
        }
    });
}

eeb_status eeb_debug_gemm(eeb_ctx* c, int tier, int dtype, int n, int k, int batch, int mode, const void* w_host,
                          const void* x_host, float* y_host) {
    return guarded([&] {
        if (!c || !w_host || !x_host || !y_host) throw Error(EEB_E_DOMAIN, "null argument");
        if (n <= 0 || k <= 0 || batch <= 0 || batch > 1024 || (mode != 0 && mode != 2 && mode != 3) ||
            (mode == 3 && n % 2))
            throw Error(EEB_E_DOMAIN, "bad gemm shape or mode");
        EEB_CUDA(cudaSetDevice(c->device));
        const size_t es = dtype == EEB_BF16 ? 2 : 4;
        const int n_out = mode == 3 ? n / 2 : n;
        DevBuf w, x, act, ws, na;
        w.ensure((size_t)n * k * es);
        x.ensure((size_t)batch * k * es);
        act.ensure((size_t)batch * n_out * es);
        const int64_t plane = (int64_t)batch * n;
        const int max_planes = std::max(k / 128 + 2, c->num_sms + 1);
        ws.ensure((size_t)plane * max_planes * 4);
        na.ensure(4);
        EEB_CUDA(cudaMemcpy(w.p, w_host, w.bytes, cudaMemcpyHostToDevice));
        EEB_CUDA(cudaMemcpy(x.p, x_host, x.bytes, cudaMemcpyHostToDevice));
        EEB_CUDA(cudaMemcpy(na.p, &batch, 4, cudaMemcpyHostToDevice));
        GemmArgs a;
        a.dtype = dtype; a.W = w.p; a.X = x.p; a.n_active = na.as<int>(); a.max_rows = batch; a.N = n; a.K = k;
        a.out = ws.as<float>(); a.plane_stride = plane; a.max_planes = max_planes; a.num_sms = c->num_sms;
        if (tier == 2 && mode != 0 && dtype == EEB_BF16) {  // the step's path: activation fused in the epilogue
            a.act_out = act.p;
            a.act_kind = mode == 3 ? 2 : 1;
            a.out = nullptr;
            a.max_planes = 1;
        }
        const int planes = tier == 2 ? gemm_tc(a, c->stream) : gemm_cc(a, c->stream);
        if (planes == 0) throw Error(EEB_E_DOMAIN, "tensor-core tier not applicable");
        if (mode == 0) {  // fixed-order sum of the planes on the host
            std::vector<float> tmp((size_t)plane * planes);
            EEB_CUDA(cudaStreamSynchronize(c->stream));
            EEB_CUDA(cudaMemcpy(tmp.data(), ws.p, tmp.size() * 4, cudaMemcpyDeviceToHost));
            for (int64_t i = 0; i < plane; ++i) {
                float v = 0.f;
                for (int p2 = 0; p2 < planes; ++p2) v += tmp[(size_t)p2 * plane + i];
                y_host[i] = v;
            }
            return;
        }
        if (!a.act_out)
            launch_act(dtype, ws.as<float>(), planes, plane, na.as<int>(), batch, n, mode == 3, act.p, c->num_sms,
                       c->stream);
        EEB_CUDA(cudaStreamSynchronize(c->stream));
        std::vector<char> tmp((size_t)batch * n_out * es);
        EEB_CUDA(cudaMemcpy(tmp.data(), act.p, tmp.size(), cudaMemcpyDeviceToHost));
        for (size_t i = 0; i < (size_t)batch * n_out; ++i) {
            if (es == 4) std::memcpy(&y_host[i], &tmp[i * 4], 4);
            else {
                uint16_t h;
                std::memcpy(&h, &tmp[i * 2], 2);
                const uint32_t u = (uint32_t)h << 16;
                std::memcpy(&y_host[i], &u, 4);
            }
        }
    });
}

eeb_status eeb_debug_bench_gemm(eeb_ctx* c, int tier, int n, int k, int batch, int iters, double* ms_out) {
    return guarded([&] {
        if (!c || !ms_out || n <= 0 || k <= 0 || batch <= 0 || iters <= 0) throw Error(EEB_E_DOMAIN, "bad argument");
        EEB_CUDA(cudaSetDevice(c->device));
        // Rotate over enough distinct weight copies (>= 512 MB, 4x L2) that every
        // launch streams its weights from HBM, as in the step.
        DevBuf x, ws, na;
        const size_t wbytes = (size_t)n * k * 2;
        const int nbuf = std::getenv("EEB_BENCH_L2") ? 1 : (int)std::max<size_t>(1, ((size_t)512 << 20) / wbytes + 1);
        std::vector<std::unique_ptr<DevBuf>> wv;
        for (int i = 0; i < nbuf; ++i) {
            wv.push_back(std::make_unique<DevBuf>());
            wv.back()->ensure(wbytes);
            synth_linear(EEB_BF16, wv.back()->p, 1 + i, 1, n, k, 0.02f, false, k, c->stream);
        }
        x.ensure((size_t)batch * k * 2);
        const int64_t plane = (int64_t)batch * n;
        const int max_planes = std::max(k / 128 + 2, c->num_sms + 1);
        ws.ensure((size_t)plane * max_planes * 4);
        na.ensure(4);
        synth_linear(EEB_BF16, x.p, 2, 1, batch, k, 1.0f, false, k, c->stream);
        EEB_CUDA(cudaMemcpy(na.p, &batch, 4, cudaMemcpyHostToDevice));
        GemmArgs a;
        a.dtype = EEB_BF16; a.W = wv[0]->p; a.X = x.p; a.n_active = na.as<int>(); a.max_rows = batch; a.N = n; a.K = k;
        a.out = ws.as<float>(); a.plane_stride = plane; a.max_planes = max_planes; a.num_sms = c->num_sms;
        // EEB_BENCH_ACT=1 (ReLU) / 2 (SwiGLU): the fused up projection (4-CTA
        // cluster K reduction + activation epilogue) as layer_core launches it
        static const int bench_act = std::getenv("EEB_BENCH_ACT") ? std::atoi(std::getenv("EEB_BENCH_ACT")) : 0;
        DevBuf act;
        if (bench_act) {
            act.ensure((size_t)batch * n * 2);
            a.out = nullptr;
            a.plane_stride = 0;
            a.max_planes = 1;
            a.act_out = act.p;
            a.act_kind = bench_act;
        }
        int it = 0;
        static const bool bench_pf = std::getenv("EEB_BENCH_PF") != nullptr;  // + L2 prefetch of the next copy
        auto run = [&] {
            a.W = wv[it++ % nbuf]->p;
            if (bench_pf) {
                a.pf = wv[it % nbuf]->p;
                a.pf_bytes = wbytes;
            }
            if (tier == 2) {
                if (gemm_tc(a, c->stream) == 0) throw Error(EEB_E_DOMAIN, "tensor-core tier not applicable");
            } else {
                gemm_cc(a, c->stream);
            }
        };
        for (int i = 0; i < 3; ++i) run();
        cudaEvent_t e0, e1;
        EEB_CUDA(cudaEventCreate(&e0));
        EEB_CUDA(cudaEventCreate(&e1));
        EEB_CUDA(cudaEventRecord(e0, c->stream));
        // EEB_GEMM_TRACE=path: globaltimer stamps of every CTA of two consecutive
        // mid-chain launches (u64 [2][ctas][8]) written to path
        static const char* trace_path = std::getenv("EEB_GEMM_TRACE");
        DevBuf trace;
        const size_t tr_per = (size_t)8 * 2048;
        if (trace_path) {
            trace.ensure(2 * tr_per * 8);
            EEB_CUDA(cudaMemset(trace.p, 0, 2 * tr_per * 8));
        }
        for (int i = 0; i < iters; ++i) {
            a.trace = trace_path && (i == iters / 2 || i == iters / 2 + 1)
                          ? trace.as<unsigned long long>() + (i - iters / 2) * tr_per : nullptr;
            run();
        }
        a.trace = nullptr;
        EEB_CUDA(cudaEventRecord(e1, c->stream));
        EEB_CUDA(cudaEventSynchronize(e1));
        float ms = 0.f;
        EEB_CUDA(cudaEventElapsedTime(&ms, e0, e1));
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        *ms_out = ms / iters;
        if (trace_path) {
            std::vector<unsigned long long> h(2 * tr_per);
            EEB_CUDA(cudaMemcpy(h.data(), trace.p, h.size() * 8, cudaMemcpyDeviceToHost));
            if (FILE* f = std::fopen(trace_path, "wb")) {
                std::fwrite(h.data(), 8, h.size(), f);
                std::fclose(f);
            }
        }
    });
}

eeb_status eeb_profile_enable(eeb_ctx* c, int enable) {
    return guarded([&] {
        if (!c) throw Error(EEB_E_DOMAIN, "null context");
        c->profiling = enable ? 1 : 0;
        for (int k = 0; k < kNumCat; ++k) { c->cat_ms[k] = 0; c->cat_launches[k] = 0; }
        c->steps_profiled = 0;
    });
}

eeb_status eeb_profile_read(eeb_ctx* c, char* json_out, int64_t cap) {
    return guarded([&] {
        if (!c || !json_out) throw Error(EEB_E_DOMAIN, "null argument");
        std::string j = "{\"steps\": " + std::to_string(c->steps_profiled) + ", \"last_step_launches\": " +
                        std::to_string(c->step_launches);
        for (int k = 0; k < kNumCat; ++k) {
            char buf[160];
            std::snprintf(buf, sizeof buf, ", \"%s_ms\": %.6f, \"%s_launches\": %lld", kCatNames[k], c->cat_ms[k],
                          kCatNames[k], (long long)c->cat_launches[k]);
            j += buf;
        }
        j += "}";
        if ((int64_t)j.size() + 1 > cap) throw Error(EEB_E_DOMAIN, "buffer too small");
        std::memcpy(json_out, j.c_str(), j.size() + 1);
    });
}

void* eeb_stream(eeb_ctx* c) { return c ? (void*)c->stream : nullptr; }

eeb_status eeb_tp_px_alloc(eeb_ctx* c, int model, void** dev_ptr, uint8_t* ipc_handle64) {
    return guarded([&] {
        if (!c) throw Error(EEB_E_DOMAIN, "null context");
        Model& m = model_of(c, model);
        if (m.tp < 2 || m.rank < 0)
            throw Error(EEB_E_DOMAIN, "peer exchange needs a tensor-parallel rank model (tp_size >= 2, tp_rank >= 0)");
        if (m.tp > kPxMaxRanks) throw Error(EEB_E_DOMAIN, "peer exchange supports at most 8 ranks");
        EEB_CUDA(cudaSetDevice(c->device));
        const PxLayout L = px_layout(m);
        if (m.px.bytes < (size_t)L.bytes) {
            m.px.release();
            m.px.ensure((size_t)L.bytes);
        }
        EEB_CUDA(cudaMemset(m.px.p, 0, m.px.bytes));
        if (dev_ptr) *dev_ptr = m.px.p;
        if (ipc_handle64) {
            cudaIpcMemHandle_t h;
            EEB_CUDA(cudaIpcGetMemHandle(&h, m.px.p));
            static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
            std::memcpy(ipc_handle64, &h, 64);
        }
    });
}

eeb_status eeb_tp_px_attach(eeb_ctx* c, int model, int nranks, void* const* peer_ptrs, const uint8_t* ipc_handles64) {
    return guarded([&] {
        if (!c) throw Error(EEB_E_DOMAIN, "null context");
        Model& m = model_of(c, model);
        if (!m.px.p) throw Error(EEB_E_STALE, "eeb_tp_px_alloc first");
        if (nranks != m.tp) throw Error(EEB_E_DOMAIN, "nranks must equal the model's tp_size");
        if (!peer_ptrs && !ipc_handles64) throw Error(EEB_E_DOMAIN, "peer pointers or IPC handles required");
        EEB_CUDA(cudaSetDevice(c->device));
        cudaDeviceSynchronize();
        for (void* q : m.px_opened) cudaIpcCloseMemHandle(q);
        m.px_opened.clear();
        PxPeers P;
        P.nranks = nranks;
        P.rank = m.rank;
        P.lay = px_layout(m);
        for (int p = 0; p < nranks; ++p) {
            if (p == m.rank) {
                P.base[p] = static_cast<char*>(m.px.p);
            } else if (peer_ptrs && peer_ptrs[p]) {
                // a buffer of this process: same device, or a peer GPU over NVLink
                cudaPointerAttributes at{};
                EEB_CUDA(cudaPointerGetAttributes(&at, peer_ptrs[p]));
                if (at.device != c->device) {
                    const cudaError_t e = cudaDeviceEnablePeerAccess(at.device, 0);
                    if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
                    else EEB_CUDA(e);
                }
                P.base[p] = static_cast<char*>(peer_ptrs[p]);
            } else {
                cudaIpcMemHandle_t h;
                std::memcpy(&h, ipc_handles64 + (size_t)p * 64, 64);
                void* q = nullptr;
                EEB_CUDA(cudaIpcOpenMemHandle(&q, h, cudaIpcMemLazyEnablePeerAccess));
                m.px_opened.push_back(q);
                P.base[p] = static_cast<char*>(q);
            }
        }
        m.pxp = P;
        drop_graphs(c, model);  // captured steps hold the exchange pointers by value
    });
}

eeb_status eeb_nccl_unique_id(uint8_t* id128) {
    return guarded([&] {
        ncclUniqueId id;
        if (nccl().get_unique_id(&id) != ncclSuccess) throw Error(EEB_E_CUDA, "ncclGetUniqueId failed");
        std::memcpy(id128, id.internal, 128);
    });
}

eeb_status eeb_nccl_init(eeb_ctx* c, const uint8_t* id128, int nranks, int rank) {
    return guarded([&] {
        if (!c || !id128) throw Error(EEB_E_DOMAIN, "null argument");
        EEB_CUDA(cudaSetDevice(c->device));
        ncclUniqueId id;
        std::memcpy(id.internal, id128, 128);
        ncclResult_t r = nccl().comm_init_rank(&c->nccl, nranks, id, rank);
        if (r != ncclSuccess) throw Error(EEB_E_CUDA, std::string("ncclCommInitRank: ") + nccl().error_string(r));
    });
}

eeb_status eeb_profile_allreduce(eeb_ctx* c, int64_t* counters, int n, double* sum_neg_logprob) {
    return guarded([&] {
        if (!c || !c->nccl) throw Error(EEB_E_STALE, "NCCL communicator not initialised");
        if (n < 0 || (n > 0 && !counters)) throw Error(EEB_E_DOMAIN, "bad counter array");
        c->nccl_buf.ensure((size_t)n * 8 + 8);
        int64_t* dc = c->nccl_buf.as<int64_t>();
        double* dd = reinterpret_cast<double*>(dc + n);
        if (n) EEB_CUDA(cudaMemcpyAsync(dc, counters, (size_t)n * 8, cudaMemcpyHostToDevice, c->stream));
        if (sum_neg_logprob) EEB_CUDA(cudaMemcpyAsync(dd, sum_neg_logprob, 8, cudaMemcpyHostToDevice, c->stream));
        const NcclApi& api = nccl();
        api.group_start();
        if (n) api.all_reduce(dc, dc, n, ncclInt64, ncclSum, c->nccl, c->stream);
        if (sum_neg_logprob) api.all_reduce(dd, dd, 1, ncclFloat64, ncclSum, c->nccl, c->stream);
        ncclResult_t r = api.group_end();
        if (r != ncclSuccess) throw Error(EEB_E_CUDA, std::string("ncclAllReduce: ") + api.error_string(r));
        if (n) EEB_CUDA(cudaMemcpyAsync(counters, dc, (size_t)n * 8, cudaMemcpyDeviceToHost, c->stream));
        if (sum_neg_logprob) EEB_CUDA(cudaMemcpyAsync(sum_neg_logprob, dd, 8, cudaMemcpyDeviceToHost, c->stream));
        EEB_CUDA(cudaStreamSynchronize(c->stream));
    });
}

}  // extern "C"
