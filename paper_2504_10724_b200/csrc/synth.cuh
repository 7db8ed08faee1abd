// synth.cuh — definition of the synthetic early-exit decoder's weights.
//
// There are no checkpoints (no network), so every weight is a pure function of
// (model seed, tensor id, flat element index) through a counter-based hash.
// The same definition is restated independently in oracle/eeb_oracle.c; the
// two agree bit-for-bit because each element is computed with exactly two
// correctly-rounded f32 multiplies (no FMA contraction on either side).
//
// "Biased exit heads" (BASELINE north star; SURVEY §7 hard part 3): the
// residual stream's first half is a reserved subspace carrying, for input
// token t, a(t)·G(t,·) with a(t) = A·(1 − z(t)) and z(t) ~ U[0,1) seeded per
// token.  Layers never write it (the o_proj / down_proj rows of that half are
// zero), so it reaches every exit head unchanged.  Head e reads it through
// α_e·G(σ(v),·) for vocabulary row v, which puts a logit of size
// α_e·a(t)·(d/2)/rms on token v* = σ⁻¹(t) and Gaussian noise elsewhere.  α_e is
// solved in closed form so that a token is confident (>= design_th) at head e
// exactly when z(t) <= coverage_e: the exit distribution over uniformly drawn
// tokens reproduces the stated cumulative coverage, e.g. 73.0 / 4.7 / 22.3 %
// at layers 6 / 12 / 24 (fixtures/FIXTURES.md:47-55).
#pragma once

#include <stdint.h>

#include <cmath>
#include <vector>

#ifndef EEB_HD
#if defined(__CUDACC__)
#define EEB_HD __host__ __device__ __forceinline__
#else
#define EEB_HD inline
#endif
#endif

namespace eeb {
namespace synth {

// Tensor kinds.  Layer tensors: id = layer * 16 + kind (layer 1-indexed).
enum LayerTensor : int {
    kAttnNorm = 0,
    kWqkv = 1,
    kWo = 2,
    kMlpNorm = 3,
    kWup = 4,   // relu: [F, d]; swiglu: [2F, d] with rows (2j, 2j+1) = (gate_j, up_j)
    kWdown = 5,
};
// Base tensors: id = 8192 + kind * 64 + exit index.
enum BaseTensor : int {
    kEmbG = 0,       // unit-variance table G shared by embedding and heads
    kZ = 1,          // per-token difficulty z(t)
    kHeadNoise = 2,  // per-head independent noise R_e
    kHeadNorm = 3,   // per-head RMSNorm gain
};

EEB_HD int layer_tid(int layer, int kind) { return layer * 16 + kind; }
EEB_HD int base_tid(int kind, int e) { return 8192 + kind * 64 + e; }

constexpr float kUnit = 3.46410161513775f;  // 2*sqrt(3): U(-1/2,1/2) * kUnit has unit variance
constexpr float kSigma = 0.02f;             // N(0, 0.02^2)-scale init of the non-residual projections
constexpr float kA = 0.25f;                 // max amplitude of the reserved (signal) half
constexpr float kB = 1.0f;                  // amplitude of the free half of the embedding
constexpr float kBeta = 0.02f;              // per-head independent noise
constexpr float kNormJitter = 0.1f;         // RMSNorm gains are 1 + U(-0.1, 0.1)
constexpr double kLayerVar = 2e-3;          // target per-layer residual variance added (free half)
constexpr uint32_t kPermMul = 7919u;        // σ(v) = (v * P + 17) mod V, P coprime to V
constexpr uint32_t kPermAdd = 17u;

EEB_HD uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

// Uniform in [-1/2, 1/2) with 24 bits (exactly representable in f32).
EEB_HD float hash_uniform(uint64_t seed, int tid, uint64_t idx) {
    uint64_t h = mix64(seed + 0x9E3779B97F4A7C15ULL * (uint64_t)(tid + 1));
    h = mix64(h ^ (idx * 0xD1B54A32D192ED03ULL + 0x632BE59BD9B4E019ULL));
    const uint32_t u = (uint32_t)(h >> 40);
    return (float)u * 5.9604644775390625e-08f - 0.5f;  // u * 2^-24 - 1/2, exact
}

#if defined(__CUDA_ARCH__)
EEB_HD float mul_rn(float a, float b) { return __fmul_rn(a, b); }
EEB_HD float add_rn(float a, float b) { return __fadd_rn(a, b); }
#else
EEB_HD float mul_rn(float a, float b) { return a * b; }  // host TU compiled with -ffp-contract=off
EEB_HD float add_rn(float a, float b) { return a + b; }
#endif

// Unit-variance draw.
EEB_HD float unit(uint64_t seed, int tid, uint64_t idx) {
    return mul_rn(hash_uniform(seed, tid, idx), kUnit);
}

EEB_HD float z_of(uint64_t seed, int token) {
    return hash_uniform(seed, base_tid(kZ, 0), (uint64_t)token) + 0.5f;  // [0, 1)
}
EEB_HD float amp_of(uint64_t seed, int token) {
    return mul_rn(kA, 1.0f - z_of(seed, token));  // 1 - z exact in f32 (24-bit z)
}

EEB_HD uint32_t perm_mul(uint32_t vocab) {
    uint32_t p = kPermMul;
    for (;;) {  // smallest p >= 7919 coprime to vocab
        uint32_t a = p, b = vocab;
        while (b) { uint32_t t = a % b; a = b; b = t; }
        if (a == 1) return p;
        ++p;
    }
}
EEB_HD int sigma_of(int v, uint32_t vocab, uint32_t pmul) {
    return (int)(((uint64_t)v * pmul + kPermAdd) % vocab);
}

// Embedding row t, element i.
EEB_HD float emb_value(uint64_t seed, int d, int t, int i) {
    const float g = unit(seed, base_tid(kEmbG, 0), (uint64_t)t * d + i);
    return mul_rn(g, i < d / 2 ? amp_of(seed, t) : kB);
}

// Head e, vocabulary row v, element i.
EEB_HD float head_value(uint64_t seed, int d, int e, float alpha_e, int v, int i, uint32_t vocab,
                        uint32_t pmul) {
    const float noise = mul_rn(unit(seed, base_tid(kHeadNoise, e), (uint64_t)v * d + i), kBeta);
    if (i >= d / 2) return noise;
    const int src = sigma_of(v, vocab, pmul);
    const float sig = mul_rn(unit(seed, base_tid(kEmbG, 0), (uint64_t)src * d + i), alpha_e);
    return add_rn(sig, noise);
}

EEB_HD float norm_gain(uint64_t seed, int tid, int i) {
    return add_rn(1.0f, mul_rn(hash_uniform(seed, tid, (uint64_t)i), 2.0f * kNormJitter));
}

// Residual-projection scale: per-layer added variance ~kLayerVar on the free half.
inline float residual_sigma(int d, int ffn) {
    const double var_h = (double)d * kSigma * kSigma / 2.0;  // E[relu(u)^2] per hidden unit
    return (float)std::sqrt(kLayerVar / ((double)ffn * var_h));
}

// Linear-layer element: row r of an [rows, cols] matrix.
// zero_signal_rows: o_proj / down_proj do not write the reserved half.
EEB_HD float linear_value(uint64_t seed, int tid, int r, int c, int cols, float scale,
                          bool zero_signal_rows, int d) {
    if (zero_signal_rows && r < d / 2) return 0.0f;
    return mul_rn(unit(seed, tid, (uint64_t)r * cols + c), scale);
}

// Closed-form head gains.  At the boundary amplitude a* = A(1 - c_e) the
// target logit minus the log-sum-exp of the other V-1 logits must equal
// logit(th).  With k = alpha * a*/rms the target is k*d/2 and the others are
// ~N(0, k^2 d/2 + beta^2 d) (lse = ln(V-1) + var/2), giving
// k = 1 - sqrt(1 - 4C/d), C = ln(V-1) + beta^2 d / 2 + logit(th).
inline std::vector<float> head_alphas(int d, int vocab, int num_layers,
                                      const std::vector<int>& exit_layers,
                                      const std::vector<float>& coverage, float th) {
    std::vector<float> out;
    const double thc = th <= 0.0f ? 1e-6 : (th >= 1.0f ? 1.0 - 1e-6 : (double)th);
    const double C = std::log((double)vocab - 1.0) + (double)kBeta * kBeta * d / 2.0 +
                     std::log(thc / (1.0 - thc));
    double disc = 1.0 - 4.0 * C / d;
    if (disc < 0.05) disc = 0.05;
    const double k = 1.0 - std::sqrt(disc);
    for (size_t e = 0; e < exit_layers.size(); ++e) {
        double c = coverage[e];
        if (c > 0.99) c = 0.99;
        if (c < 0.01) c = 0.01;
        const double a_star = (double)kA * (1.0 - c);
        const double n2 = kLayerVar * exit_layers[e];  // free-half variance added by the layers
        const double rms = std::sqrt((a_star * a_star + (double)kB * kB + n2) / 2.0);
        out.push_back((float)(k * rms / a_star));
    }
    (void)num_layers;
    return out;
}

}  // namespace synth
}  // namespace eeb
