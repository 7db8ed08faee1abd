// exit_head.cu — exit-head reduction (K2 tail), exit decisions, survivor
// compaction (K3) and the exit-layer histogram (K4).
//
// Reference semantics reproduced here (all in /root/reference/proj/include/eeserve):
//   confidence  = max softmax probability, logprob = log-prob of the emitted
//                 (argmax) token — SPEC.md:106, ExitObservation trace.hpp:17-22;
//   argmax ties → lowest token id (pinned here; the reference has no logits);
//   introspective exit: first head with confidence >= th, final head forced —
//                 earliest_confident_obs trace.hpp:69-76;
//   flat:       the head at the serving depth (or the deepest head below it),
//                 exit_layer = depth — observation_for_depth trace.hpp:86-97,
//                 engine.hpp:350-354;
//   breached   = confidence < th (strict) — engine.hpp:353,358; false at full depth (:363);
//   unchanged  = head token == final token — engine.hpp:366;
//   histogram  = ExitHistogram::add per exit layer — pht.hpp:19-22, engine.hpp:49.
#include "../../include/eeb/eeb.h"
#include <algorithm>

#include "kernels.h"

namespace eeb {

namespace {

constexpr int kReduceThreads = 1024;

// Per-row max / argmax / sum-exp over the vocabulary.
__global__ void __launch_bounds__(kReduceThreads)
    head_reduce_kernel(Stamp stamp, const float* part, int splits, int64_t split_stride, int vocab,
                       const int* n_active, HeadOut h, float* logits_out) {
    StampScope stamp_scope(stamp);
    pdl_launch_dependents();
    pdl_wait();
    const int i = blockIdx.x;
    if (i >= *n_active) return;
    extern __shared__ float lg[];  // [vocab] summed logits of this row
    const float* l = lg;
    float m = -INFINITY;
    int am = 0x7fffffff;
    for (int v = threadIdx.x; v < vocab; v += kReduceThreads) {
        float x = 0.f;
        for (int s = 0; s < splits; ++s) x += part[s * split_stride + (int64_t)i * vocab + v];
        lg[v] = x;
        if (logits_out) logits_out[(int64_t)i * vocab + v] = x;
        if (x > m) { m = x; am = v; }  // strided scan: first occurrence within the thread
    }
    __shared__ float ms[32];
    __shared__ int as[32];
    __shared__ float ss[32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const float m2 = __shfl_xor_sync(0xffffffffu, m, o);
        const int a2 = __shfl_xor_sync(0xffffffffu, am, o);
        if (m2 > m || (m2 == m && a2 < am)) { m = m2; am = a2; }
    }
    if (lane == 0) { ms[warp] = m; as[warp] = am; }
    __syncthreads();
    if (warp == 0) {
        m = ms[lane];
        am = as[lane];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const float m2 = __shfl_xor_sync(0xffffffffu, m, o);
            const int a2 = __shfl_xor_sync(0xffffffffu, am, o);
            if (m2 > m || (m2 == m && a2 < am)) { m = m2; am = a2; }
        }
        if (lane == 0) { ms[0] = m; as[0] = am; }
    }
    __syncthreads();
    const float mx = ms[0];
    float s = 0.f;
    for (int v = threadIdx.x; v < vocab; v += kReduceThreads) s += __expf(l[v] - mx);
    s = warp_sum(s);
    if (lane == 0) ss[warp] = s;
    __syncthreads();
    if (warp == 0) {
        s = warp_sum(ss[lane]);
        if (lane == 0) {
            h.tok[i] = as[0];
            h.conf[i] = 1.0f / s;
            h.logp[i] = -logf(s);
        }
    }
}

__device__ __forceinline__ void write_row(const StepOutDev& o, int r, int exit_layer, int tok,
                                          float conf, float logp, int breached, int unchanged,
                                          int bin) {
    o.exit_layer[r] = exit_layer;
    o.token_id[r] = tok;
    o.confidence[r] = conf;
    o.logprob[r] = logp;
    o.breached[r] = (uint8_t)breached;
    o.unchanged[r] = (uint8_t)unchanged;
    o.bin[r] = bin;
}

// Applies the token policy to the rows the head just ran on and, for
// introspective steps, compacts the survivors (ballot + block scan).  With the
// fused head the per-tile partials are merged first, a warp per row spread
// over the grid (one SM's L2 bandwidth would bound a single-CTA merge); the
// last CTA to finish (ticket) then decides for every row.
constexpr int kDecideThreads = 256;
__global__ void __launch_bounds__(kDecideThreads) decide_kernel(Stamp stamp, DecideArgs a) {
    StampScope stamp_scope(stamp);
    pdl_launch_dependents();
    pdl_wait();
    stamp_waited(stamp);
    __shared__ int warp_counts[32];
    __shared__ int n_live_s;
    __shared__ int last_s;
    const int n_live = *a.cur.n_active;
    const int e = a.exit_index;
    if (a.head_tri) {
        // K2 tail of the fused head GEMM: merge the per-(row, vocab tile)
        // {max, sum exp, argmax} partials — warp per row, tiles in a fixed
        // order (deterministic); argmax ties resolve to the lowest token id.
        const int lane = threadIdx.x & 31, nw = blockDim.x >> 5;
        const int tiles = a.head_tiles * a.head_shards;
        for (int i = blockIdx.x * nw + (threadIdx.x >> 5); i < n_live; i += gridDim.x * nw) {
            const float4* tri = reinterpret_cast<const float4*>(a.head_tri) + (int64_t)i * a.head_tiles;
            // tile t of the whole vocabulary: region t / head_tiles (a TP shard), local tile t % head_tiles
            auto at = [&](int t) {
                const int r = t / a.head_tiles;
                return tri[r * a.head_shard_stride + (t - r * a.head_tiles)];
            };
            // kPre partials per lane are loaded at once (one L2 latency per
            // chunk, not one per tile); same per-lane order as a strided scan
            // (measured: holding all 16 per lane in registers for a single
            // round of loads is ~1 us slower per decide)
            constexpr int kPre = 8;
            float m = -INFINITY;
            int am = 0x7fffffff;
            for (int t0 = lane; t0 < tiles; t0 += 32 * kPre) {
                float4 pre[kPre];
#pragma unroll
                for (int k = 0; k < kPre; ++k)
                    pre[k] = t0 + 32 * k < tiles ? at(t0 + 32 * k)
                                                 : make_float4(-INFINITY, 0.f, __int_as_float(0x7fffffff), 0.f);
#pragma unroll
                for (int k = 0; k < kPre; ++k) {
                    const int ai = __float_as_int(pre[k].z);
                    if (pre[k].x > m || (pre[k].x == m && ai < am)) { m = pre[k].x; am = ai; }
                }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const float m2 = __shfl_xor_sync(0xffffffffu, m, o);
                const int a2 = __shfl_xor_sync(0xffffffffu, am, o);
                if (m2 > m || (m2 == m && a2 < am)) { m = m2; am = a2; }
            }
            float sum = 0.f;
            for (int t0 = lane; t0 < tiles; t0 += 32 * kPre) {
                float4 pre[kPre];
#pragma unroll
                for (int k = 0; k < kPre; ++k)
                    pre[k] = t0 + 32 * k < tiles ? at(t0 + 32 * k) : make_float4(-INFINITY, 0.f, 0.f, 0.f);
#pragma unroll
                for (int k = 0; k < kPre; ++k)
                    if (t0 + 32 * k < tiles) sum += pre[k].y * __expf(pre[k].x - m);
            }
            sum = warp_sum(sum);
            if (lane == 0) {
                a.head.tok[i] = am;
                a.head.conf[i] = 1.0f / sum;
                a.head.logp[i] = -logf(sum);
            }
        }
        if (gridDim.x > 1) {
            __threadfence();  // this CTA's merged rows, visible before its ticket
            __syncthreads();
            if (threadIdx.x == 0) last_s = atomicAdd(a.ticket, 1) == (int)gridDim.x - 1;
            __syncthreads();
            if (!last_s) return;
            __threadfence();
            if (threadIdx.x == 0) *a.ticket = 0;  // every CTA has arrived: ready for the next launch
        }
        __syncthreads();
    }
    const StepOutDev& o = a.out;
    int survivors_total = 0;
    for (int base = 0; base < n_live; base += blockDim.x) {
        const int i = base + threadIdx.x;
        const bool live = i < n_live;
        bool survive = false;
        if (live) {
            const int r = a.cur.row_of[i];
            const int tok = a.head.tok[i];
            const float conf = a.head.conf[i];
            const float logp = a.head.logp[i];
            switch (a.policy) {
                case EEB_FLAT:
                    write_row(o, r, a.serving_depth, tok, conf, logp, conf < a.th,
                              a.is_final && a.exit_layer == a.num_layers ? 1 : 2, e);
                    break;
                case EEB_FULL_DEPTH:
                    write_row(o, r, a.num_layers, tok, conf, logp, 0, 1, e);
                    break;
                case EEB_INTROSPECTIVE:
                    if (a.is_final) {
                        write_row(o, r, a.exit_layer, tok, conf, logp, conf < a.th, 1, e);
                    } else if (conf >= a.th) {
                        write_row(o, r, a.exit_layer, tok, conf, logp, 0, 2, e);
                    } else {
                        survive = true;
                    }
                    break;
                default: {  // EEB_PROFILE: record every head, decide at the final one
                    o.head_token[(int64_t)r * a.n_exits + e] = tok;
                    o.head_confidence[(int64_t)r * a.n_exits + e] = conf;
                    o.head_logprob[(int64_t)r * a.n_exits + e] = logp;
                    if (a.is_final) {
                        int ex = a.n_exits - 1;
                        for (int k = 0; k < a.n_exits; ++k)
                            if (o.head_confidence[(int64_t)r * a.n_exits + k] >= a.th) { ex = k; break; }
                        const int64_t q = (int64_t)r * a.n_exits + ex;
                        write_row(o, r, a.layers[ex], o.head_token[q], o.head_confidence[q],
                                  o.head_logprob[q], o.head_confidence[q] < a.th,
                                  o.head_token[q] == tok ? 1 : 0, ex);
                    }
                    break;
                }
            }
        }
        if (a.policy != EEB_INTROSPECTIVE || a.is_final) continue;
        // K3: warp ballot + block exclusive scan of survivors.
        const unsigned ballot = __ballot_sync(0xffffffffu, survive);
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        if (lane == 0) warp_counts[warp] = __popc(ballot);
        __syncthreads();
        if (threadIdx.x == 0) {
            int run = 0;
            for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
                const int c = warp_counts[w];
                warp_counts[w] = run;
                run += c;
            }
            n_live_s = run;
        }
        __syncthreads();
        if (survive) {
            const int j = survivors_total + warp_counts[warp] + __popc(ballot & ((1u << lane) - 1u));
            a.gather_src[j] = i;
            a.nxt.row_of[j] = a.cur.row_of[i];
            a.nxt.slot[j] = a.cur.slot[i];
            a.nxt.pos[j] = a.cur.pos[i];
        }
        survivors_total += n_live_s;
        __syncthreads();
    }
    if (a.policy == EEB_INTROSPECTIVE && !a.is_final && threadIdx.x == 0) {
        *a.nxt.n_active = survivors_total;
        // no survivor: the deeper layers' conditional body is skipped
        if (a.has_cond) cudaGraphSetConditional(a.cond, survivors_total > 0 ? 1u : 0u);
    }
}

// K4 + bookkeeping: shared-memory atomic histogram of exit-head bins, breach
// count, fixed-order f64 logprob sum, KV depth map update.
__global__ void __launch_bounds__(1024)
    finalize_kernel(Stamp stamp, int batch, int n_exits, StepOutDev o, const int* slot_in,
                    const int* pos_in, uint8_t* kv_depth, int max_seq,
                    int computed_depth) {
    StampScope stamp_scope(stamp);
    pdl_launch_dependents();
    pdl_wait();
    __shared__ unsigned long long hist_s[64];
    __shared__ int breach_s;
    if (threadIdx.x < 64) hist_s[threadIdx.x] = 0;
    if (threadIdx.x == 0) breach_s = 0;
    __syncthreads();
    int my_breach = 0;
    for (int r = threadIdx.x; r < batch; r += blockDim.x) {
        const int b = o.bin[r];
        if (b >= 0 && b < n_exits) atomicAdd(&hist_s[b], 1ull);
        my_breach += o.breached[r] ? 1 : 0;
        // layers whose K/V this step wrote for the row: its exit layer, or every
        // layer in the profiling pass (all heads at full depth)
        kv_depth[(int64_t)slot_in[r] * max_seq + pos_in[r]] =
            (uint8_t)(computed_depth > 0 ? computed_depth : o.exit_layer[r]);
    }
    atomicAdd(&breach_s, my_breach);
    __syncthreads();
    if (threadIdx.x < n_exits) o.hist[threadIdx.x] = (int64_t)hist_s[threadIdx.x];
    // fixed row order: deterministic and batch-order defined (the rows' log
    // probs staged in smem by one parallel load, summed by one thread)
    __shared__ float lp_s[1024];
    const bool staged = batch <= 1024;
    if (staged)
        for (int r = threadIdx.x; r < batch; r += blockDim.x) lp_s[r] = o.logprob[r];
    __syncthreads();
    if (threadIdx.x == 0) {
        *o.n_breached = breach_s;
        double s = 0.0;
        for (int r = 0; r < batch; ++r) s += (double)(staged ? lp_s[r] : o.logprob[r]);
        *o.sum_logprob = s;
    }
}

}  // namespace

void launch_head_reduce(const float* part, int splits, int64_t split_stride, int vocab, const int* n_active,
                        int max_rows, HeadOut h, float* logits_out, cudaStream_t s) {
    const size_t smem = (size_t)vocab * 4;
    if (smem > 200 * 1024) throw Error(1, "head_reduce: vocabulary above 51200 entries");
    EEB_CUDA(cudaFuncSetAttribute(head_reduce_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    launch_pdl(head_reduce_kernel, dim3(max_rows), dim3(kReduceThreads), smem, s, part, splits, split_stride, vocab,
               n_active, h, logits_out);
    EEB_CHECK_LAUNCH();
}

void launch_decide(const DecideArgs& a, cudaStream_t s) {
    const int warps = kDecideThreads / 32;
    const int grid = a.head_tri && a.ticket ? std::max(1, (a.max_rows + warps - 1) / warps) : 1;
    launch_pdl(decide_kernel, dim3(grid), dim3(kDecideThreads), 0, s, a);
    EEB_CHECK_LAUNCH();
}

void launch_finalize(int batch, int n_exits, StepOutDev out, const int* slot_in, const int* pos_in,
                     uint8_t* kv_depth, int max_seq, int computed_depth, cudaStream_t s) {
    if (n_exits > 64) throw Error(1, "finalize: at most 64 exits");
    launch_pdl(finalize_kernel, dim3(1), dim3(1024), 0, s, batch, n_exits, out, slot_in, pos_in, kv_depth, max_seq,
               computed_depth);
    EEB_CHECK_LAUNCH();
}

}  // namespace eeb
