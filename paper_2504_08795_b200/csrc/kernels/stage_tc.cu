// Persistent stage kernel: one launch runs a whole DARIS stage (a DNN
// segment between two synchronisation points) on the SMs of its
// partition.
//
// A stage is a chain of layers (conv on tcgen05, plus the CUDA-core pack /
// pool / depthwise / linear layers). Every layer is cut into work units
// (conv: 128 x 64 output tile x K split). CTAs claim units from one global
// atomic counter in topological (layer) order; a unit of layer l starts its
// activation reads once layer l-1 has published all of its tiles (a per-layer
// completion counter). Because a unit is only ever claimed by a running CTA
// and only waits on units claimed before it, the earliest unfinished unit can
// always run: the scheme needs no co-residency guarantee, so stage kernels of
// different tenants may share SMs (OS > 1) in any mix without deadlock.
//
// Per CTA (192 threads):
//   warp 4    scheduler: claims units, publishes them through a 2-deep smem
//             queue, and streams each conv unit's weight tiles by TMA before
//             the unit's inputs exist (weights are constant).
//   warps 0-3 wait for the layer dependency, gather activations with cp.async
//             straight into the 128B-swizzled UMMA layout, then run the fused
//             epilogue (TMEM -> scale/bias/residual/act -> bf16 NHWC); they
//             also execute the CUDA-core layers.
//   warp 5    one thread issues tcgen05.mma (128 x 64 x 16) into a 64-column
//             TMEM accumulator.
// Split-K partials are reduced with red.global.add.v4.f32 into an fp32 tile;
// the split that arrives last (atomic ticket) reads the sum, re-zeroes it and
// runs the epilogue — nobody waits for anybody.
//
// Reads of data produced inside the kernel go through L2 only (cp.async.cg,
// ld.global.cg): L1 is not coherent across SMs within one launch.
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>
#include "sm100.cuh"
#include "../../../include/daris_kernels.h"

namespace daris {
namespace stage {

constexpr int kBM = 128;
constexpr int kBN = 64;
constexpr int kBK = 64;
constexpr int kStages = 3;
constexpr int kQueue = 1;
constexpr int kThreads = 192;
constexpr int kMaxLayers = 64;
constexpr int kABytes = kBM * 128;
constexpr int kBBytes = kBN * 128;
constexpr int kTmemCols = 64;

enum Kind : int { CONV = 0, PACK8 = 1, MAXPOOL = 2, AVGPOOL = 3, LINEAR = 4, DWCONV = 5 };

// Division by a layer-invariant divisor as multiply-high + shift (n < 2^31):
// runtime integer division is a ~20-instruction dependent chain, and the
// gather computes a dozen of them per unit on the critical path.
struct FDiv {
  uint32_t mul, shr;  // mul == 0: divisor 1
};
__host__ inline FDiv make_fdiv(int d) {
  FDiv f{0, 0};
  if (d <= 1) return f;
  int l = 0;
  while ((1u << l) < static_cast<uint32_t>(d)) ++l;  // ceil(log2 d)
  const uint64_t p = 31 + l;
  f.mul = static_cast<uint32_t>(((1ull << p) + d - 1) / d);
  f.shr = static_cast<uint32_t>(p - 32);
  return f;
}
__device__ __forceinline__ int fdiv(int n, FDiv d) {
  return d.mul ? static_cast<int>(__umulhi(static_cast<uint32_t>(n), d.mul) >> d.shr) : n;
}

struct Layer {
  int kind, units, unit_begin, done_target;
  int relu, map_idx, flags, items_per_unit;
  const void* x;
  void* y;
  const __nv_bfloat16* res;
  const void* w;
  const float* scale;
  const float* bias;
  int n, h, w_, c, cout, kh, kw, stride, pad, ho, wo, M;
  int num_kb, kb_per_split, splits, cin_blocks, tiles_n, tiles;
  FDiv d_howo, d_wo, d_kw, d_cinb, d_splits, d_tilesn;
};

struct Prog {
  const Layer* layers;
  const CUtensorMap* maps;
  int* ctrs;    // [0] claim, [1] exit, [2 .. 2+L) per-layer done, [2+L ..) split-K tile tickets
  float* ws;    // split-K accumulators (zero; re-zeroed by each tile's finaliser)
  unsigned long long* trace;  // optional: 8 globaltimer stamps per unit (profiling), or null
  int n_layers, total_units;
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define STAMP(u, k)                                                        \
  do {                                                                     \
    if (P.trace) P.trace[16ull * (u) + (k)] = gtimer();                     \
  } while (0)

struct Smem {
  static constexpr int kAOff = 0;
  static constexpr int kBOff = kStages * kABytes;
  static constexpr int kBarOff = kBOff + kStages * kBBytes;
  // full[S], empty[S], tmem_full, tmem_empty, uq_full[Q], uq_empty[Q]
  static constexpr int kNumBars = 2 * kStages + 2 + 2 * kQueue;
  static constexpr int kMiscOff = kBarOff + 8 * kNumBars;        // tmem slot, flag, queue ints
  static constexpr int kEpiOff = kMiscOff + 64;                   // folded-BN scale/bias of the unit's 64 columns
  static constexpr int kTotal = kEpiOff + 2 * kBN * 4 + 1024;     // 3 CTAs fit one SM
};

__device__ __forceinline__ float act_apply(float v, int relu) {
  if (relu == 1) return fmaxf(v, 0.f);
  if (relu == 6) return fminf(fmaxf(v, 0.f), 6.f);
  return v;
}

__device__ __forceinline__ uint4 ldcg16(const void* p) { return __ldcg(reinterpret_cast<const uint4*>(p)); }

__device__ __forceinline__ void unpack8(uint4 v, float* f) {
  const uint32_t vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const float2 t = unpack_bf16x2(vv[e]);
    f[2 * e] = t.x;
    f[2 * e + 1] = t.y;
  }
}
__device__ __forceinline__ uint4 pack8(const float* f) {
  uint4 pk;
  pk.x = pack_bf16x2(f[0], f[1]);
  pk.y = pack_bf16x2(f[2], f[3]);
  pk.z = pack_bf16x2(f[4], f[5]);
  pk.w = pack_bf16x2(f[6], f[7]);
  return pk;
}

// 32 accumulator columns of one output row -> scale/bias/residual/act -> bf16
__device__ __forceinline__ void finalize_row32(const Layer& L, int m, int col0, const float* v) {
  const float4* sc = reinterpret_cast<const float4*>(L.scale + col0);
  const float4* bi = reinterpret_cast<const float4*>(L.bias + col0);
  float o[32];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const float4 s = __ldg(sc + q), b = __ldg(bi + q);
    o[4 * q + 0] = v[4 * q + 0] * s.x + b.x;
    o[4 * q + 1] = v[4 * q + 1] * s.y + b.y;
    o[4 * q + 2] = v[4 * q + 2] * s.z + b.z;
    o[4 * q + 3] = v[4 * q + 3] * s.w + b.w;
  }
  const size_t off = static_cast<size_t>(m) * L.cout + col0;
  if (L.res != nullptr) {
    uint4 r[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) r[q] = ldcg16(L.res + off + 8 * q);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      float f[8];
      unpack8(r[q], f);
#pragma unroll
      for (int e = 0; e < 8; ++e) o[8 * q + e] += f[e];
    }
  }
  uint4* yp = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(L.y) + off);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    float f[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) f[e] = act_apply(o[8 * q + e], L.relu);
    yp[q] = pack8(f);
  }
}

// publish: one release reduction (covers this CTA's writes ordered before it by bar.sync)
__device__ __forceinline__ void red_release_add(int* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void producers_sync() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

__device__ __forceinline__ int ld_relaxed_gpu(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// Spin on a completion counter with relaxed loads (an acquire load invalidates
// the SM's whole L1 on every poll), then one acquire fence.
__device__ __forceinline__ void wait_counter(const int* p, int target) {
  if (ld_relaxed_gpu(p) < target) {
    const unsigned long long t0 = gtimer();
    while (ld_relaxed_gpu(p) < target) {
      // a dependency that is not met within 2 s means a corrupted program
      // (e.g. one program launched twice concurrently): fail loudly, never hang
      if (gtimer() - t0 > 2000000000ull) __trap();
    }
  }
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
}

// ------------------------------------------------------------- CUDA-core layers
// All run on warps 0-3 (128 threads), one unit = `items_per_unit` items.
__device__ void run_pack8(const Layer& L, int unit, int tid) {
  // fp32 NCHW [n][c][h][w] -> bf16 NHWC [n][h][w][8] (c <= 8), one item = one pixel
  const float* x = static_cast<const float*>(L.x);
  uint4* y = static_cast<uint4*>(L.y);
  const int hw = L.h * L.w_;
  const int total = L.n * hw;
  const int b = unit * L.items_per_unit;
  const int e = min(total, b + L.items_per_unit);
  for (int i = b + tid; i < e; i += 128) {
    const int img = i / hw, p = i - img * hw;
    float f[8];
#pragma unroll
    for (int ci = 0; ci < 8; ++ci) f[ci] = ci < L.c ? __ldg(x + (static_cast<size_t>(img) * L.c + ci) * hw + p) : 0.f;
    y[i] = pack8(f);
  }
}

__device__ void run_maxpool(const Layer& L, int unit, int tid) {
  const __nv_bfloat16* x = static_cast<const __nv_bfloat16*>(L.x);
  uint4* y = static_cast<uint4*>(L.y);
  const int chunks = L.c / 8;
  const int total = L.n * L.ho * L.wo * chunks;
  const int b = unit * L.items_per_unit;
  const int e = min(total, b + L.items_per_unit);
  for (int i = b + tid; i < e; i += 128) {
    const int ch = i % chunks;
    const int m = i / chunks;
    const int ow = m % L.wo, oh = (m / L.wo) % L.ho, img = m / (L.wo * L.ho);
    float best[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) best[q] = -INFINITY;
    for (int r = 0; r < L.kh; ++r) {
      const int ih = oh * L.stride - L.pad + r;
      if (ih < 0 || ih >= L.h) continue;
      for (int s = 0; s < L.kw; ++s) {
        const int iw = ow * L.stride - L.pad + s;
        if (iw < 0 || iw >= L.w_) continue;
        float f[8];
        unpack8(ldcg16(x + ((static_cast<size_t>(img) * L.h + ih) * L.w_ + iw) * L.c + ch * 8), f);
#pragma unroll
        for (int q = 0; q < 8; ++q) best[q] = fmaxf(best[q], f[q]);
      }
    }
    y[i] = pack8(best);
  }
}

__device__ void run_dwconv(const Layer& L, int unit, int tid) {
  const __nv_bfloat16* x = static_cast<const __nv_bfloat16*>(L.x);
  const __nv_bfloat16* wt = static_cast<const __nv_bfloat16*>(L.w);
  uint4* y = static_cast<uint4*>(L.y);
  const int chunks = L.c / 8;
  const int total = L.n * L.ho * L.wo * chunks;
  const int b = unit * L.items_per_unit;
  const int e = min(total, b + L.items_per_unit);
  for (int i = b + tid; i < e; i += 128) {
    const int ch = i % chunks;
    const int m = i / chunks;
    const int ow = m % L.wo, oh = (m / L.wo) % L.ho, img = m / (L.wo * L.ho);
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int r = 0; r < L.kh; ++r) {
      const int ih = oh * L.stride - L.pad + r;
      if (ih < 0 || ih >= L.h) continue;
      for (int s = 0; s < L.kw; ++s) {
        const int iw = ow * L.stride - L.pad + s;
        if (iw < 0 || iw >= L.w_) continue;
        float a[8], q[8];
        unpack8(ldcg16(x + ((static_cast<size_t>(img) * L.h + ih) * L.w_ + iw) * L.c + ch * 8), a);
        unpack8(__ldg(reinterpret_cast<const uint4*>(wt + static_cast<size_t>(r * L.kw + s) * L.c) + ch), q);
#pragma unroll
        for (int k = 0; k < 8; ++k) acc[k] = fmaf(a[k], q[k], acc[k]);
      }
    }
    float o[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) o[k] = act_apply(acc[k] * __ldg(L.scale + ch * 8 + k) + __ldg(L.bias + ch * 8 + k), L.relu);
    y[i] = pack8(o);
  }
}

__device__ void run_avgpool(const Layer& L, int unit, int tid) {
  // NHWC bf16 [n][h*w][c] -> fp32 [n][c]; one item = (image, 8 channels)
  const __nv_bfloat16* x = static_cast<const __nv_bfloat16*>(L.x);
  float* y = static_cast<float*>(L.y);
  const int chunks = L.c / 8;
  const int hw = L.h * L.w_;
  const int total = L.n * chunks;
  const int b = unit * L.items_per_unit;
  const int e = min(total, b + L.items_per_unit);
  for (int i = b + tid; i < e; i += 128) {
    const int img = i / chunks, ch = i - img * chunks;
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const __nv_bfloat16* px = x + static_cast<size_t>(img) * hw * L.c + ch * 8;
#pragma unroll 7
    for (int p = 0; p < hw; ++p) {
      float f[8];
      unpack8(ldcg16(px + static_cast<size_t>(p) * L.c), f);
#pragma unroll
      for (int k = 0; k < 8; ++k) acc[k] += f[k];
    }
    const float inv = 1.f / static_cast<float>(hw);
    float4* dst = reinterpret_cast<float4*>(y + static_cast<size_t>(img) * L.c + ch * 8);
    dst[0] = make_float4(acc[0] * inv, acc[1] * inv, acc[2] * inv, acc[3] * inv);
    dst[1] = make_float4(acc[4] * inv, acc[5] * inv, acc[6] * inv, acc[7] * inv);
  }
}

__device__ void run_linear(const Layer& L, int unit, int tid) {
  // y[b][o] = act(x[b] . w[o] + bias[o]); x fp32 (flags&1: bf16), y fp32 (flags&2: bf16)
  // one unit = items_per_unit outputs, one warp per output at a time
  const int warp = tid >> 5, lane = tid & 31;
  const __nv_bfloat16* w = static_cast<const __nv_bfloat16*>(L.w);
  const int K = L.c, O = L.cout;
  const int o_begin = unit * L.items_per_unit;
  const int o_end = min(O, o_begin + L.items_per_unit);
  for (int o = o_begin + warp; o < o_end; o += 4) {
    const __nv_bfloat16* wr = w + static_cast<size_t>(o) * K;
    for (int b = 0; b < L.n; ++b) {
      float acc = 0.f;
      for (int k = lane * 8; k < K; k += 256) {
        float wf[8], xf[8];
        unpack8(__ldg(reinterpret_cast<const uint4*>(wr + k)), wf);
        if (L.flags & 1) {
          unpack8(ldcg16(static_cast<const __nv_bfloat16*>(L.x) + static_cast<size_t>(b) * K + k), xf);
        } else {
          const float4* px = reinterpret_cast<const float4*>(static_cast<const float*>(L.x) + static_cast<size_t>(b) * K + k);
          const float4 p0 = __ldcg(px), p1 = __ldcg(px + 1);
          xf[0] = p0.x; xf[1] = p0.y; xf[2] = p0.z; xf[3] = p0.w;
          xf[4] = p1.x; xf[5] = p1.y; xf[6] = p1.z; xf[7] = p1.w;
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) acc = fmaf(wf[q], xf[q], acc);
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
      if (lane == 0) {
        float v = act_apply(acc + (L.bias ? __ldg(L.bias + o) : 0.f), L.relu);
        const size_t oi = static_cast<size_t>(b) * O + o;
        if (L.flags & 2) static_cast<__nv_bfloat16*>(L.y)[oi] = __float2bfloat16_rn(v);
        else static_cast<float*>(L.y)[oi] = v;
      }
    }
  }
}

__device__ __forceinline__ int find_layer(const Layer* Ls, int n_layers, int cur, int u) {
  while (cur + 1 < n_layers && u >= Ls[cur + 1].unit_begin) ++cur;
  return cur;
}

__global__ void __maxnreg__(112) stage_kernel(const __grid_constant__ Prog P) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem + Smem::kAOff;
  uint8_t* sB = smem + Smem::kBOff;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Smem::kBarOff);
  uint64_t* full = bars;
  uint64_t* empty = bars + kStages;
  uint64_t* tmem_full = bars + 2 * kStages;
  uint64_t* tmem_empty = tmem_full + 1;
  uint64_t* uq_full = tmem_full + 2;
  uint64_t* uq_empty = uq_full + kQueue;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + Smem::kMiscOff);
  int* flag = reinterpret_cast<int*>(tmem_slot + 1);
  int* uq = flag + 1;
  float* sScale = reinterpret_cast<float*>(smem + Smem::kEpiOff);
  float* sBias = sScale + kBN;
  const Layer* Ls = P.layers;  // small, read-only: stays in L1

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  int* claim = P.ctrs;
  int* exit_ctr = P.ctrs + 1;
  int* done = P.ctrs + 2;
  int* tickets = P.ctrs + 2 + P.n_layers;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 128 + 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tmem_full, 1);
    mbar_init(tmem_empty, 1);
    for (int q = 0; q < kQueue; ++q) {
      mbar_init(&uq_full[q], 1);
      mbar_init(&uq_empty[q], 2);
    }
    fence_barrier_init();
  }
  if (warp == 4) tmem_alloc<kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int n_layers = P.n_layers;
  const int total = P.total_units;

  if (warp == 4) {
    // ---------------- scheduler + weight producer ----------------
    if (lane == 0) {
      int cur = 0, kbi = 0;
      for (int q = 0;; ++q) {
        const int slot = q % kQueue;
        if (q >= kQueue) mbar_wait(&uq_empty[slot], ((q / kQueue) & 1) ^ 1);
        int u = atomicAdd(claim, 1);
        if (u >= total) u = -1;
        if (u >= 0) {
          STAMP(u, 0);
          if (P.trace) P.trace[16ull * u + 7] = blockIdx.x;
        }
        uq[slot] = u;
        mbar_arrive(&uq_full[slot]);
        if (u < 0) break;
        cur = find_layer(Ls, n_layers, cur, u);
        const Layer L = Ls[cur];  // register copy: asm memory clobbers would force re-loads
        if (L.kind != CONV) continue;
        const int local = u - L.unit_begin;
        const int tile = fdiv(local, L.d_splits), split = local - tile * L.splits;
        const int n0 = (tile - fdiv(tile, L.d_tilesn) * L.tiles_n) * kBN;
        const int kb0 = split * L.kb_per_split;
        const int nkb = min(L.num_kb, kb0 + L.kb_per_split) - kb0;
        const CUtensorMap* map = P.maps + L.map_idx;
        for (int i = 0; i < nkb; ++i, ++kbi) {
          const int s = kbi % kStages;
          if (kbi >= kStages) mbar_wait(&empty[s], ((kbi / kStages) & 1) ^ 1);
          mbar_arrive_expect_tx(&full[s], kBBytes);
          tma_load_2d(map, &full[s], sB + s * kBBytes, (kb0 + i) * kBK, n0);
        }
      }
    }
  } else if (warp == 5) {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      constexpr uint32_t idesc = umma_idesc_bf16(kBM, kBN);
      const uint32_t sA_u32 = smem_u32(sA), sB_u32 = smem_u32(sB);
      int cur = 0, kbi = 0, cu = 0;
      for (int q = 0;; ++q) {
        const int slot = q % kQueue;
        mbar_wait(&uq_full[slot], (q / kQueue) & 1);
        const int u = uq[slot];
        mbar_arrive(&uq_empty[slot]);
        if (u < 0) break;
        cur = find_layer(Ls, n_layers, cur, u);
        const Layer L = Ls[cur];
        if (L.kind != CONV) continue;
        const int local = u - L.unit_begin;
        const int split = local - fdiv(local, L.d_splits) * L.splits;
        const int kb0 = split * L.kb_per_split;
        const int nkb = min(L.num_kb, kb0 + L.kb_per_split) - kb0;
        if (cu > 0) mbar_wait(tmem_empty, (cu - 1) & 1);  // previous accumulator drained
        tc_fence_after();
        for (int i = 0; i < nkb; ++i, ++kbi) {
          const int s = kbi % kStages;
          mbar_wait(&full[s], (kbi / kStages) & 1);
          tc_fence_after();
          const uint64_t adesc = umma_desc_k_sw128(sA_u32 + s * kABytes);
          const uint64_t bdesc = umma_desc_k_sw128(sB_u32 + s * kBBytes);
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k)
            umma_bf16(tmem_base, adesc + 2 * k, bdesc + 2 * k, idesc, (i > 0 || k > 0) ? 1u : 0u);
          umma_commit(&empty[s]);
        }
        umma_commit(tmem_full);
        ++cu;
      }
    }
  } else {
    // ---------------- warps 0-3: dependencies, gather, epilogue, CUDA-core layers ----------------
    const int t = threadIdx.x;
    const int row_sub = t >> 3, chunk = t & 7;
    const uint32_t sA_u32 = smem_u32(sA);
    int cur = 0, kbi = 0, cu = 0;
    for (int q = 0;; ++q) {
      const int slot = q % kQueue;
      mbar_wait(&uq_full[slot], (q / kQueue) & 1);
      const int u = uq[slot];
      if (u < 0) break;
      cur = find_layer(Ls, n_layers, cur, u);
      const Layer L = Ls[cur];
      const int local = u - L.unit_begin;
      if (t == 0) STAMP(u, 1);
      // dependency: the previous layer of this stage has published every tile
      if (cur > 0) {
        if (t == 0) wait_counter(done + cur - 1, Ls[cur - 1].done_target);
        producers_sync();
      }
      if (t == 0) STAMP(u, 2);
      if (L.kind != CONV) {
        switch (L.kind) {
          case PACK8: run_pack8(L, local, t); break;
          case MAXPOOL: run_maxpool(L, local, t); break;
          case AVGPOOL: run_avgpool(L, local, t); break;
          case LINEAR: run_linear(L, local, t); break;
          case DWCONV: run_dwconv(L, local, t); break;
          default: break;
        }
        producers_sync();
        if (t == 0) {
          STAMP(u, 5);
          red_release_add(done + cur, 1);
          mbar_arrive(&uq_empty[slot]);  // CTA free: the scheduler may claim the next unit
        }
        continue;
      }
      // ---- conv unit ----
      const int tile = fdiv(local, L.d_splits), split = local - tile * L.splits;
      const int tile_m = fdiv(tile, L.d_tilesn), tile_n = tile - tile_m * L.tiles_n;
      const int m0 = tile_m * kBM, n0 = tile_n * kBN;
      const int kb0 = split * L.kb_per_split;
      const int nkb = min(L.num_kb, kb0 + L.kb_per_split) - kb0;
      int pix_base[8], ih0[8], iw0[8];
      const int howo = L.ho * L.wo;
#pragma unroll
      for (int p = 0; p < 8; ++p) {
        const int m = m0 + p * 16 + row_sub;
        const int img = fdiv(m, L.d_howo);
        const int rem = m - img * howo;
        const int oh = fdiv(rem, L.d_wo);
        const int ow = rem - oh * L.wo;
        const bool in = m < L.M;
        pix_base[p] = in ? img * L.h * L.w_ : 0;
        ih0[p] = in ? oh * L.stride - L.pad : -(1 << 20);  // out-of-range rows fail the bounds test
        iw0[p] = in ? ow * L.stride - L.pad : -(1 << 20);
      }
      const __nv_bfloat16* x = static_cast<const __nv_bfloat16*>(L.x);
      const bool stem = L.c == 8;
      const int ksize = L.kh * L.kw;
      constexpr int kLag = kStages - 1;
      if (t == 0) STAMP(u, 11);
      for (int i = 0; i < nkb; ++i) {
        const int s = (kbi + i) % kStages;
        if (kbi + i >= kStages) mbar_wait(&empty[s], (((kbi + i) / kStages) & 1) ^ 1);
        if (t == 0 && i == 0) STAMP(u, 12);
        const int kb = kb0 + i;
        int kpos, coff;
        if (stem) {  // stem "pixel chunks": each 16-B chunk is one kernel position's 8 channels
          kpos = kb * 8 + chunk;
          coff = 0;
        } else {
          kpos = fdiv(kb, L.d_cinb);
          coff = (kb - kpos * L.cin_blocks) * kBK + chunk * 8;
        }
        const bool kvalid = kpos < ksize;
        const int r_ = fdiv(kpos, L.d_kw), s_ = kpos - r_ * L.kw;
        const uint32_t stage_base = sA_u32 + s * kABytes;
#pragma unroll
        for (int p = 0; p < 8; ++p) {
          const int r = p * 16 + row_sub;
          const int ih = ih0[p] + r_, iw = iw0[p] + s_;
          const bool valid = kvalid && (unsigned)ih < (unsigned)L.h && (unsigned)iw < (unsigned)L.w_;
          const __nv_bfloat16* src =
              valid ? x + (static_cast<size_t>(pix_base[p] + ih * L.w_ + iw) * L.c + coff) : x;
          cp_async_16(stage_base + r * 128 + ((chunk ^ (r & 7)) << 4), src, valid);
        }
        cp_async_commit();
        if (t == 0 && i == 0) STAMP(u, 8);
        if (i >= kLag) {
          cp_async_wait<kLag>();
          fence_proxy_async_smem();
          tc_fence_before();
          mbar_arrive(&full[(kbi + i - kLag) % kStages]);
        }
      }
      // epilogue operands that do not depend on the accumulator, fetched while
      // the last loads land and the MMAs drain: folded-BN scale/bias -> smem,
      // this thread's residual row -> registers
      const float sb = t < kBN ? __ldg(L.scale + n0 + t) : __ldg(L.bias + n0 + t - kBN);
      const int row = warp * 32 + lane;
      const int m = m0 + row;
      const bool row_ok = m < L.M;
      uint4 resv[8];
      const bool has_res = L.res != nullptr && row_ok;
      if (has_res) {
        const __nv_bfloat16* rp = L.res + static_cast<size_t>(m) * L.cout + n0;
#pragma unroll
        for (int q = 0; q < 8; ++q) resv[q] = ldcg16(rp + 8 * q);
      }
      if (t == 0) STAMP(u, 9);
      cp_async_wait<0>();
      if (t == 0) STAMP(u, 10);
      fence_proxy_async_smem();
      tc_fence_before();
      for (int i = max(0, nkb - kLag); i < nkb; ++i) mbar_arrive(&full[(kbi + i) % kStages]);
      kbi += nkb;
      sScale[t] = sb;  // (sScale and sBias are contiguous: t < 64 scale, else bias)
      if (t == 0) STAMP(u, 3);

      // ---- epilogue ----
      mbar_wait(tmem_full, cu & 1);
      tc_fence_after();
      if (t == 0) {
        STAMP(u, 4);
        mbar_arrive(&uq_empty[slot]);  // MMAs retired: claim the next unit while the epilogue runs
      }
      producers_sync();  // scale/bias visible
      const uint32_t t_row = tmem_base + (static_cast<uint32_t>(warp * 32) << 16);
      __nv_bfloat16* yrow = static_cast<__nv_bfloat16*>(L.y) + static_cast<size_t>(m) * L.cout + n0;
      // v: 32 fp32 accumulator columns [c0, c0+32) of this row -> bf16 output
      auto finish32 = [&](int c0, const float* v) {
        float o[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) o[j] = v[j] * sScale[c0 + j] + sBias[c0 + j];
        if (has_res) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            float f[8];
            unpack8(resv[c0 / 8 + q], f);
#pragma unroll
            for (int e = 0; e < 8; ++e) o[8 * q + e] += f[e];
          }
        }
        uint4* yp = reinterpret_cast<uint4*>(yrow + c0);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          float f[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) f[e] = act_apply(o[8 * q + e], L.relu);
          yp[q] = pack8(f);
        }
      };
      bool publish = true;
      if (L.splits == 1) {
#pragma unroll
        for (int c0 = 0; c0 < kBN; c0 += 32) {
          uint32_t r[32];
          tmem_ld_32x32b_x32(t_row + c0, r);
          if (row_ok) finish32(c0, reinterpret_cast<const float*>(r));
        }
        tc_fence_before();
        producers_sync();
        if (t == 0) mbar_arrive(tmem_empty);
      } else {
        float* acc_row = P.ws + static_cast<size_t>(tile) * (kBM * kBN) + static_cast<size_t>(row) * kBN;
#pragma unroll 1
        for (int c0 = 0; c0 < kBN; c0 += 32) {
          uint32_t r[32];
          tmem_ld_32x32b_x32(t_row + c0, r);
          if (row_ok) {
#pragma unroll
            for (int q = 0; q < 8; ++q)
              red_add_v4(acc_row + c0 + 4 * q, __uint_as_float(r[4 * q]), __uint_as_float(r[4 * q + 1]),
                         __uint_as_float(r[4 * q + 2]), __uint_as_float(r[4 * q + 3]));
          }
        }
        tc_fence_before();
        __threadfence();
        producers_sync();
        if (t == 0) {
          mbar_arrive(tmem_empty);  // accumulator drained: the MMA warp may start the next unit
          *flag = (atomicAdd(tickets + tile, 1) == L.splits - 1);
        }
        producers_sync();
        publish = *flag != 0;
        if (publish) {
          __threadfence();
          if (row_ok) {
#pragma unroll
            for (int c0 = 0; c0 < kBN; c0 += 32) {
              float4* src = reinterpret_cast<float4*>(acc_row + c0);
              float4 part[8];
#pragma unroll
              for (int q = 0; q < 8; ++q) part[q] = __ldcg(src + q);
#pragma unroll
              for (int q = 0; q < 8; ++q) __stcg(src + q, make_float4(0.f, 0.f, 0.f, 0.f));
              finish32(c0, reinterpret_cast<const float*>(part));
            }
          }
          if (t == 0) tickets[tile] = 0;
        }
      }
      ++cu;
      if (t == 0) STAMP(u, 6);
      if (publish) {
        producers_sync();
        if (t == 0) {
          STAMP(u, 5);
          red_release_add(done + cur, 1);
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 4) {
    tc_fence_after();
    tmem_dealloc<kTmemCols>(tmem_base);
  }
  // the last CTA out re-arms the counters for the next launch of this program
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(exit_ctr, 1) == static_cast<int>(gridDim.x) - 1) {
      __threadfence();
      for (int i = 0; i < 2 + n_layers; ++i) P.ctrs[i] = 0;
      __threadfence();
    }
  }
}

}  // namespace stage
}  // namespace daris

// ------------------------------------------------------------------ host side
using namespace daris;
using namespace daris::stage;

struct daris_stage_prog {
  Prog prog{};
  Layer* d_layers = nullptr;
  CUtensorMap* d_maps = nullptr;
  int* d_ctrs = nullptr;
  float* d_ws = nullptr;
  int grid = 0;
  int n_layers = 0;
  int total_units = 0;
  int64_t ws_floats = 0;
  int n_tickets = 0;
  std::vector<Layer> layers;
};

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

static int stage_min_kb_per_split() {
  static const int v = [] {
    const char* e = std::getenv("DARIS_STAGE_MIN_KB");  // experiment knob: K blocks per split-K unit
    return e ? std::max(1, std::atoi(e)) : 2;
  }();
  return v;
}

extern "C" int daris_stage_plan_conv(const daris_stage_op* op, int32_t grid, int32_t* splits, int32_t* kb_per_split,
                                     int32_t* units) {
  if (!op || op->kind != DARIS_OP_CONV) return DARIS_K_BAD_ARG;
  const int M = op->n * op->ho * op->wo;
  const int num_kb = op->c == 8 ? (op->kh * op->kw + 7) / 8 : op->kh * op->kw * (op->c / kBK);
  const int tiles = ((M + kBM - 1) / kBM) * (op->cout / kBN);
  int s = op->splits;
  if (s <= 0) {
    s = 1;
    const int min_kb = stage_min_kb_per_split();
    if (tiles * 2 <= grid && num_kb >= 2 * min_kb) {
      s = grid / tiles;
      if (s > num_kb / min_kb) s = num_kb / min_kb;
      if (s > 16) s = 16;
      if (s < 1) s = 1;
    }
  }
  if (s > num_kb) s = num_kb;
  const int kbps = (num_kb + s - 1) / s;
  s = (num_kb + kbps - 1) / kbps;
  *splits = s;
  *kb_per_split = kbps;
  *units = tiles * s;
  return DARIS_K_OK;
}

extern "C" int daris_stage_create(const daris_stage_op* ops, int32_t n_ops, int32_t grid, daris_stage_prog** out) {
  if (!ops || n_ops < 1 || n_ops > kMaxLayers || grid < 1 || !out) return DARIS_K_BAD_ARG;
  auto encode = encode_fn();
  if (!encode) return DARIS_K_NO_DRIVER;
  auto* P = new daris_stage_prog();
  P->grid = grid;
  std::vector<CUtensorMap> maps;
  int unit = 0;
  int64_t ws = 0;
  int tickets = 0;
  for (int i = 0; i < n_ops; ++i) {
    const daris_stage_op& o = ops[i];
    Layer L{};
    L.kind = o.kind;
    L.relu = o.relu;
    L.flags = o.flags;
    L.x = o.x;
    L.y = o.y;
    L.res = static_cast<const __nv_bfloat16*>(o.residual);
    L.w = o.weight;
    L.scale = o.scale;
    L.bias = o.bias;
    L.n = o.n; L.h = o.h; L.w_ = o.w; L.c = o.c; L.cout = o.cout; L.kh = o.kh; L.kw = o.kw;
    L.stride = o.stride; L.pad = o.pad; L.ho = o.ho; L.wo = o.wo;
    L.map_idx = -1;
    bool bad = !o.x || !o.y;
    switch (o.kind) {
      case DARIS_OP_CONV: {
        if ((o.c % kBK != 0 && o.c != 8) || o.cout % kBN != 0 || !o.weight || !o.scale || !o.bias) bad = true;
        if (bad) break;
        int s = 0, kbps = 0, units = 0;
        daris_stage_plan_conv(&o, grid, &s, &kbps, &units);
        L.M = o.n * o.ho * o.wo;
        L.num_kb = o.c == 8 ? (o.kh * o.kw + 7) / 8 : o.kh * o.kw * (o.c / kBK);
        L.cin_blocks = o.c / kBK;
        L.tiles_n = o.cout / kBN;
        L.tiles = ((L.M + kBM - 1) / kBM) * L.tiles_n;
        L.splits = s;
        L.kb_per_split = kbps;
        L.d_howo = make_fdiv(o.ho * o.wo);
        L.d_wo = make_fdiv(o.wo);
        L.d_kw = make_fdiv(o.kw);
        L.d_cinb = make_fdiv(std::max(1, L.cin_blocks));
        L.d_splits = make_fdiv(s);
        L.d_tilesn = make_fdiv(L.tiles_n);
        L.units = units;
        L.done_target = L.tiles;
        if (s > 1) {
          ws = std::max<int64_t>(ws, static_cast<int64_t>(L.tiles) * kBM * kBN);
          tickets = std::max(tickets, L.tiles);
        }
        const int K = o.kh * o.kw * o.c;
        CUtensorMap map;
        cuuint64_t dims[2] = {static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(o.cout)};
        cuuint64_t strides[1] = {static_cast<cuuint64_t>(K) * 2};
        cuuint32_t box[2] = {static_cast<cuuint32_t>(kBK), static_cast<cuuint32_t>(kBN)};
        cuuint32_t estr[2] = {1, 1};
        if (encode(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(o.weight), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
          bad = true;
          break;
        }
        L.map_idx = static_cast<int>(maps.size());
        maps.push_back(map);
        break;
      }
      case DARIS_OP_PACK8: {
        if (o.c > 8) bad = true;
        L.items_per_unit = 1024;
        L.units = (o.n * o.h * o.w + L.items_per_unit - 1) / L.items_per_unit;
        break;
      }
      case DARIS_OP_MAXPOOL:
      case DARIS_OP_DWCONV: {
        if (o.c % 8 != 0) bad = true;
        if (o.kind == DARIS_OP_DWCONV && (!o.weight || !o.scale || !o.bias)) bad = true;
        L.items_per_unit = o.kind == DARIS_OP_DWCONV ? 512 : 1024;
        L.units = (o.n * o.ho * o.wo * (o.c / 8) + L.items_per_unit - 1) / L.items_per_unit;
        break;
      }
      case DARIS_OP_AVGPOOL: {
        if (o.c % 8 != 0) bad = true;
        L.items_per_unit = 128;
        L.units = (o.n * (o.c / 8) + 127) / 128;
        break;
      }
      case DARIS_OP_LINEAR: {
        if (o.c % 8 != 0 || !o.weight) bad = true;
        L.items_per_unit = 16;
        L.units = (o.cout + 15) / 16;
        break;
      }
      default:
        bad = true;
    }
    if (bad) {
      delete P;
      return DARIS_K_BAD_SHAPE;
    }
    if (o.kind != DARIS_OP_CONV) L.done_target = L.units;
    L.unit_begin = unit;
    unit += L.units;
    P->layers.push_back(L);
  }
  P->n_layers = n_ops;
  P->total_units = unit;
  P->ws_floats = ws;
  P->n_tickets = tickets;
  bool ok = cudaMalloc(&P->d_layers, sizeof(Layer) * n_ops) == cudaSuccess &&
            cudaMemcpy(P->d_layers, P->layers.data(), sizeof(Layer) * n_ops, cudaMemcpyHostToDevice) == cudaSuccess;
  if (ok && !maps.empty())
    ok = cudaMalloc(&P->d_maps, sizeof(CUtensorMap) * maps.size()) == cudaSuccess &&
         cudaMemcpy(P->d_maps, maps.data(), sizeof(CUtensorMap) * maps.size(), cudaMemcpyHostToDevice) == cudaSuccess;
  const size_t nctr = 2 + n_ops + std::max(tickets, 1);
  ok = ok && cudaMalloc(&P->d_ctrs, sizeof(int) * nctr) == cudaSuccess &&
       cudaMemset(P->d_ctrs, 0, sizeof(int) * nctr) == cudaSuccess;
  if (ok && ws > 0)
    ok = cudaMalloc(&P->d_ws, sizeof(float) * ws) == cudaSuccess &&
         cudaMemset(P->d_ws, 0, sizeof(float) * ws) == cudaSuccess;
  if (!ok) {
    daris_stage_destroy(P);
    return cudaErrorMemoryAllocation;
  }
  P->prog.layers = P->d_layers;
  P->prog.maps = P->d_maps;
  P->prog.ctrs = P->d_ctrs;
  P->prog.ws = P->d_ws;
  P->prog.n_layers = n_ops;
  P->prog.total_units = unit;
  *out = P;
  return DARIS_K_OK;
}

extern "C" int daris_stage_launch(const daris_stage_prog* P, void* stream) {
  if (!P) return DARIS_K_BAD_ARG;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(stage_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, Smem::kTotal);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  stage_kernel<<<P->grid, kThreads, Smem::kTotal, static_cast<cudaStream_t>(stream)>>>(P->prog);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int daris_stage_info(const daris_stage_prog* P, daris_stage_info_t* out) {
  if (!P || !out) return DARIS_K_BAD_ARG;
  out->grid = P->grid;
  out->layers = P->n_layers;
  out->units = P->total_units;
  out->smem_bytes = Smem::kTotal;
  out->workspace_floats = P->ws_floats;
  return DARIS_K_OK;
}

extern "C" int daris_stage_set_trace(daris_stage_prog* P, void* trace) {
  if (!P) return DARIS_K_BAD_ARG;
  P->prog.trace = static_cast<unsigned long long*>(trace);
  return DARIS_K_OK;
}

extern "C" int daris_stage_layer_units(const daris_stage_prog* P, int32_t layer, int32_t* units, int32_t* splits) {
  if (!P || layer < 0 || layer >= P->n_layers) return DARIS_K_BAD_ARG;
  *units = P->layers[layer].units;
  *splits = P->layers[layer].kind == CONV ? P->layers[layer].splits : 1;
  return DARIS_K_OK;
}

extern "C" void daris_stage_destroy(daris_stage_prog* P) {
  if (!P) return;
  if (P->d_layers) cudaFree(P->d_layers);
  if (P->d_maps) cudaFree(P->d_maps);
  if (P->d_ctrs) cudaFree(P->d_ctrs);
  if (P->d_ws) cudaFree(P->d_ws);
  delete P;
}
