// Implicit-GEMM convolution on the sm_100a tensor cores (tcgen05 + TMEM + TMA).
//
// GEMM view: M = n*ho*wo output pixels, N = cout, K = kh*kw*cin with K ordered
// (kh, kw, cin) so one 64-wide K block is 64 contiguous NHWC channels of one
// input pixel (128 B). Per CTA: a 128 x BN output tile, fp32 accumulator in
// TMEM (BN columns), a STAGES-deep smem ring of (activation, weight) K blocks.
//
// conv_igemm_tc_kernel (one CTA per tile, up to 3 CTAs per SM at 96 registers):
//   warps 0-3  epilogue (and, for shapes TMA cannot box — 224-wide VGG rows,
//              8-channel stems without the padded layout — the activation
//              gather: cp.async of 128 rows x 128 B straight into the 128B-
//              swizzled UMMA layout)
//   warp 4     TMA producer: weights as 2-D boxes {64, BN}; activations as a
//              4-D box of th whole output rows traversed with the conv stride
//              (padding = TMA zero fill), the stem's overlapping 128-B windows,
//              or the fused downsample branch; the residual tile into a ring
//              stage the K loop leaves free (RT); owns TMEM
//   warp 5     MMA issuer: one thread, 4 x tcgen05.mma (K = 16) per K block
// Epilogue: TMEM -> registers -> folded-BN scale/bias, residual, ReLU(6) ->
// bf16 staged 128B-swizzled in the idle ring -> TMA store.
// Split-K (small-M layers at batch 1): inside a cluster of <= 8 CTAs every
// split stages its fp32 partial in its idle ring and, after one cluster
// barrier, each CTA pulls its share of the valid rows from all peers over DSMEM
// and runs the epilogue; without clusters, red.global.add into a zeroed tile +
// a ticket for the last arriver, which re-zeroes both for the next launch.
//
// conv_pair_kernel (large-M launches): a (2,1,1) cluster runs one UMMA M = 256
// tile on tcgen05.mma.cta_group::2 — see its comment below.
//
// Programmatic dependent launch: weights do not depend on the previous layer,
// so the TMA warp starts streaming them before griddepcontrol.wait; the
// activation producers wait, and every CTA triggers its dependents as soon as
// its mainloop is done so the next layer's prologue overlaps this epilogue.
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <mutex>
#include "sm100.cuh"
#include "../../../include/daris_kernels.h"

namespace daris {

constexpr int kBM = 128;
constexpr int kBK = 64;            // bf16 elements per K block = 128 B rows
constexpr int kThreads = 192;
// Register cap of the conv kernels. Registers are split over the SM's four
// sub-partitions (16K each) and a 6-warp CTA puts 2 warps on two of them: at
// 112 regs/thread a sub-partition holds 4 warps -> 2 CTAs per SM; at 96 it
// holds 5 -> 3 CTAs per SM (shared memory allows 3 at BN <= 128). ptxas spills
// 16 B at 96 (a stack slot in L1).
#ifndef DARIS_CONV_MAXNREG
#define DARIS_CONV_MAXNREG 96
#endif
// Pipeline depth per tile width: shallow rings keep smem per CTA small so three
// CTAs (of different tenants' kernels) fit on one SM — at batch 1 the layers
// are latency-bound and co-residency, not pipeline depth, sets throughput.
#ifndef DARIS_BN64_STAGES
#define DARIS_BN64_STAGES 3
#endif
template <int BN> struct Depth { static constexpr int kStages = DARIS_BN64_STAGES; };
template <> struct Depth<128> { static constexpr int kStages = 2; };
template <> struct Depth<256> { static constexpr int kStages = 2; };

// Division by a launch-invariant divisor as multiply-high + shift (n < 2^31):
// a runtime integer division is a ~20-instruction dependent chain and the
// activation gather needs a dozen of them before its first load.
struct FDiv {
  uint32_t mul, shr;  // mul == 0: divisor 1
};
static inline FDiv make_fdiv(int d) {
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

struct ConvArgs {
  const __nv_bfloat16* x;
  __nv_bfloat16* y;
  const __nv_bfloat16* res;
  const float* scale;
  const float* bias;
  float* ws;
  int* counters;
  int n, h, w, cin, cout, kh, kw, stride, pad, ho, wo;
  int M, relu, num_kb, kb_per_split, splits, cin_blocks;
  int cluster_split;  // 1: the splits of a tile form one cluster and reduce through DSMEM
  int tma_a;          // 1: activations arrive by TMA (4-D box = th whole output rows of one image)
  int th, tiles_h;    // TMA mode: output rows per M tile, M tiles per image
  int ipt;            // TMA mode with th == ho: whole images per M tile (the boxes' image extent)
  int tma_c;          // 1: the epilogue stages the bf16 tile in smem and stores it with TMA (splits == 1)
  int res_tma;        // 1: the residual tile arrives by TMA into the ring stage the K loop never uses
  int stem_tma;       // 1: 8-channel stem from a zero-bordered input, one TMA window box per kernel row
  int kb_seg1;        // K blocks of the primary input; blocks >= kb_seg1 come from x2 (DARIS_CONV_DUAL)
  int stride2;        // x2 sampling stride
  int box_rows;       // rows of one output/residual TMA box
  unsigned long long* ts;  // optional per-CTA phase timestamps (globaltimer ns), 16 per CTA
  FDiv d_howo, d_wo, d_kw, d_cinb, d_tiles_h;
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

template <int BN, int ST = Depth<BN>::kStages>
struct SmemLayout {
  static constexpr int kStages = ST;
  static constexpr int kLag = kStages - 1;  // cp.async groups kept in flight per producer thread
  static constexpr int kABytes = kBM * 128;
  static constexpr int kBBytes = BN * 128;
  static constexpr int kAOff = 0;
  static constexpr int kBOff = kStages * kABytes;
  static constexpr int kBarOff = kBOff + kStages * kBBytes;
  static constexpr int kEpiOff = kBarOff + 256;         // folded-BN scale[BN], bias[BN] of this tile
  static constexpr int kTotal = kEpiOff + 2 * BN * 4 + 1024;  // + alignment slack
};

__device__ __forceinline__ uint4 ldg_nc16(const void* p) { return __ldg(reinterpret_cast<const uint4*>(p)); }

// 32 accumulator columns of one output row -> scale/bias (smem) -> bf16, then
// the residual add and the activation on packed bf16 pairs -> 4 x 16 B. The
// residual is added after rounding acc*scale+bias to bf16 (one extra bf16
// rounding, <= 0.5 ulp): unpacking the residual to fp32, adding and
// activating per element was ~60 % of the epilogue's instructions, and the
// epilogue sets the memory-bound layers' time (ResNet-50 b64: see DESIGN §3).
__device__ __forceinline__ void pack_row32(const ConvArgs& a, int c_local, const float* v, const float* s_scale,
                                           const float* s_bias, const uint4 (&res4)[4], bool use_res,
                                           uint4 (&pk)[4]) {
  // scale/bias as 16-B smem vectors (c_local is a multiple of 32: aligned)
  const float4* sc4 = reinterpret_cast<const float4*>(s_scale + c_local);
  const float4* bi4 = reinterpret_cast<const float4*>(s_bias + c_local);
  __nv_bfloat162 h[16];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const float4 sc = sc4[q], bi = bi4[q];
    h[2 * q] = __floats2bfloat162_rn(fmaf(v[4 * q + 0], sc.x, bi.x), fmaf(v[4 * q + 1], sc.y, bi.y));
    h[2 * q + 1] = __floats2bfloat162_rn(fmaf(v[4 * q + 2], sc.z, bi.z), fmaf(v[4 * q + 3], sc.w, bi.w));
  }
  if (use_res) {
    const __nv_bfloat162* r2 = reinterpret_cast<const __nv_bfloat162*>(res4);
#pragma unroll
    for (int i = 0; i < 16; ++i) h[i] = __hadd2(h[i], r2[i]);
  }
  // one uniform branch per 32 columns (the activation chosen per element
  // compiled to a uniform compare + branch around every element)
  if (a.relu == 1) {
    const __nv_bfloat162 z = __float2bfloat162_rn(0.f);
#pragma unroll
    for (int i = 0; i < 16; ++i) h[i] = __hmax2(h[i], z);
  } else if (a.relu == 6) {
    const __nv_bfloat162 z = __float2bfloat162_rn(0.f), six = __float2bfloat162_rn(6.f);
#pragma unroll
    for (int i = 0; i < 16; ++i) h[i] = __hmin2(__hmax2(h[i], z), six);
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) pk[q] = *reinterpret_cast<const uint4*>(&h[4 * q]);
}

// ... and straight to this row of the NHWC output (one thread per row).
__device__ __forceinline__ void finalize_row32(const ConvArgs& a, int m, int col0, int c_local, const float* v,
                                               const float* s_scale, const float* s_bias, const uint4 (&res4)[4],
                                               bool use_res) {
  uint4 pk[4];
  pack_row32(a, c_local, v, s_scale, s_bias, res4, use_res, pk);
  uint4* yp = reinterpret_cast<uint4*>(a.y + static_cast<size_t>(m) * a.cout + col0);
#pragma unroll
  for (int q = 0; q < 4; ++q) yp[q] = pk[q];
}

#ifdef DARIS_PAIR_DEBUG
// Debug build only: a pair-kernel mbarrier wait that has not completed after 2 s
// records (site, rank, block) into host-mapped memory (daris_debug_pair_watch)
// and keeps waiting, so a host watchdog can read where a hung launch sits.
__device__ unsigned int* g_pair_watch = nullptr;
__device__ __forceinline__ bool mbar_try(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ void pair_wait(uint64_t* bar, uint32_t parity, int site) {
  const unsigned long long t0 = gtimer();
  bool reported = false;
  while (!mbar_try(bar, parity)) {
    if (!reported && gtimer() - t0 > 2000000000ull && g_pair_watch) {
      reported = true;
      const unsigned int i = atomicAdd(g_pair_watch, 1u);
      if (i < 60)
        g_pair_watch[4 + i] = static_cast<unsigned int>(site) | (cluster_rank() << 4) | (parity << 5) |
                              (blockIdx.x << 8) | (blockIdx.y << 20);
      __threadfence_system();
    }
  }
}
#define PAIR_WAIT(bar, parity, site) pair_wait(bar, parity, site)
// in-flight counters (host-mapped words 32..47): +1 entering / -1 leaving a blocking op
#define DBG_IN(k) do { if (g_pair_watch) atomicAdd(g_pair_watch + 32 + (k), 1u); } while (0)
#define DBG_OUT(k) do { if (g_pair_watch) atomicSub(g_pair_watch + 32 + (k), 1u); } while (0)
#else
#define PAIR_WAIT(bar, parity, site) mbar_wait(bar, parity)
#define DBG_IN(k) do {} while (0)
#define DBG_OUT(k) do {} while (0)
#endif

template <int BN, int ST, bool RT = false>  // RT: the residual tile arrives by TMA (ConvArgs::res_tma)
__global__ void __maxnreg__(DARIS_CONV_MAXNREG)
    conv_igemm_tc_kernel(const __grid_constant__ CUtensorMap wmap, const __grid_constant__ CUtensorMap amap,
                         const __grid_constant__ CUtensorMap ymap, const __grid_constant__ CUtensorMap amap2,
                         const __grid_constant__ CUtensorMap rmap, const ConvArgs a) {
  using L = SmemLayout<BN, ST>;
  constexpr int kStages = L::kStages;
  constexpr int kLag = L::kLag;
  extern __shared__ uint8_t smem_raw[];
  // 1024-B aligned by pointer arithmetic on smem_raw (an integer round trip would
  // lose the shared address space: every smem access would become a generic LD/ST)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem + L::kAOff;
  uint8_t* sB = smem + L::kBOff;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::kBarOff);
  uint64_t* empty = full + kStages;
  uint64_t* tmem_full = empty + kStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);
  int* last_flag = reinterpret_cast<int*>(tmem_slot + 1);
  uint64_t* res_bar = tmem_full + 2;  // the residual tile has landed (res_tma)

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int tile_m = blockIdx.x, tile_n = blockIdx.y, split = blockIdx.z;
  unsigned long long* ts = a.ts ? a.ts + 16ull * (blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z)) : nullptr;
  if (ts && threadIdx.x == 0) {
    ts[0] = gtimer();
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    ts[15] = smid;
  }
  // M tile -> first output pixel m0 and number of valid rows. Gather mode: 128
  // consecutive flattened pixels. TMA mode: th whole output rows of one image
  // (th * wo <= 128 rows; the rest of the 128-row MMA tile is ignored).
  int m0, mvalid, img = 0, h0 = 0;
  if (a.tma_a) {
    const int q = fdiv(tile_m, a.d_tiles_h);
    img = q * a.ipt;
    h0 = (tile_m - q * a.tiles_h) * a.th;
    m0 = img * (a.ho * a.wo) + h0 * a.wo;
    mvalid = min(a.th, a.ho - h0) * a.wo * min(a.ipt, a.n - img);
  } else {
    m0 = tile_m * kBM;
    mvalid = min(kBM, a.M - m0);
  }
  const int n0 = tile_n * BN;
  const int kb_begin = split * a.kb_per_split;
  const int kb_end = min(a.num_kb, kb_begin + a.kb_per_split);
  const int nkb = kb_end - kb_begin;
  // RT: residual half h (64 channels x 128 rows, 128B-swizzled like the output
  // staging) in ring stage rs — A slot for h = 0, B slot for h = 1 (BN = 128) —
  // the stage K block nkb would take: unused by a K loop shorter than the ring,
  // else the first stage the MMAs free (its load overlaps the last K blocks).
  // Output staging: the bf16 halves in stage st (A slot, then B slot at BN = 128),
  // clear of the residual; contiguous from A stage 0 without RT.
  const int rs = nkb % kStages;
  const int st_stage = RT ? (rs + 1) % kStages : 0;
  uint8_t* res_half0 = sA + rs * L::kABytes;
  uint8_t* res_half1 = sB + rs * L::kBBytes;
  auto out_half = [&](int h) -> uint8_t* {
    return (BN == 128 && h == 1) ? sB + st_stage * L::kBBytes : sA + st_stage * L::kABytes + h * (kBM * 128);
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], a.tma_a ? 1 : 128 + 1);  // TMA mode: one expect_tx arrival covers A and B
      mbar_init(&empty[s], 1);
    }
    mbar_init(tmem_full, 1);
    mbar_init(res_bar, 1);
    fence_barrier_init();
  }
  if (warp == 4) {
    if (lane == 0) DBG_IN(4);
    tmem_alloc<BN>(tmem_slot);
    if (lane == 0) DBG_OUT(4);
    if (lane == 0) {
      tma_prefetch_desc(&wmap);
      if (a.tma_a) tma_prefetch_desc(&amap);
      if (a.tma_c) tma_prefetch_desc(&ymap);
      if (a.kb_seg1 < a.num_kb) tma_prefetch_desc(&amap2);
      if (RT) tma_prefetch_desc(&rmap);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (ts && threadIdx.x == 0) ts[1] = gtimer();

  if (warp < 4) {
    // ---------------- activation producer (gather mode) + epilogue ----------------
    const int t = threadIdx.x;
    const int row_sub = t >> 3, chunk = t & 7;
    float* s_scale = reinterpret_cast<float*>(smem + L::kEpiOff);
    float* s_bias = s_scale + BN;
    // folded-BN scale/bias of this tile -> smem (constant: loaded before the dependency wait)
    for (int c = t; c < BN; c += 128) {
      s_scale[c] = __ldg(a.scale + n0 + c);
      s_bias[c] = __ldg(a.bias + n0 + c);
    }
    if (a.tma_a) {
      pdl_wait();  // the residual below comes from an earlier layer
      if (ts && threadIdx.x == 0) ts[2] = gtimer();
    } else {
    int pix_base[8], ih0[8], iw0[8];
    const int howo = a.ho * a.wo;
#pragma unroll
    for (int p = 0; p < 8; ++p) {
      const int m = m0 + p * 16 + row_sub;
      const int im = fdiv(m, a.d_howo);
      const int rem = m - im * howo;
      const int oh = fdiv(rem, a.d_wo);
      const int ow = rem - oh * a.wo;
      const bool in = m < a.M;
      pix_base[p] = in ? im * a.h * a.w : 0;
      ih0[p] = in ? oh * a.stride - a.pad : -(1 << 20);  // out-of-range rows fail the bounds test
      iw0[p] = in ? ow * a.stride - a.pad : -(1 << 20);
    }
    const bool stem = a.cin == 8;
    const int ksize = a.kh * a.kw;
    pdl_wait();  // activations come from the previous layer
    if (ts && threadIdx.x == 0) ts[2] = gtimer();
    const uint32_t sA_u32 = smem_u32(sA);
    for (int i = 0; i < nkb; ++i) {
      const int s = i % kStages;
      if (i >= kStages) mbar_wait(&empty[s], ((i / kStages) & 1) ^ 1);
      const int kb = kb_begin + i;
      // K block -> (kernel position, channel offset) of this thread's 16-B chunk.
      // Normal layers: one position per K block, 64 channels. Stem layers
      // (cin == 8, "pixel chunks"): every chunk is one position's 8 channels.
      int kpos, coff;
      if (stem) {
        kpos = kb * 8 + chunk;
        coff = 0;
      } else {
        kpos = fdiv(kb, a.d_cinb);
        coff = (kb - kpos * a.cin_blocks) * kBK + chunk * 8;
      }
      const bool kvalid = kpos < ksize;
      const int r_ = fdiv(kpos, a.d_kw), s_ = kpos - r_ * a.kw;
      const uint32_t stage_base = sA_u32 + s * L::kABytes;
#pragma unroll
      for (int p = 0; p < 8; ++p) {
        const int r = p * 16 + row_sub;
        const int ih = ih0[p] + r_, iw = iw0[p] + s_;
        const bool valid = kvalid && (unsigned)ih < (unsigned)a.h && (unsigned)iw < (unsigned)a.w;
        const __nv_bfloat16* src =
            valid ? a.x + (static_cast<size_t>(pix_base[p] + ih * a.w + iw) * a.cin + coff) : a.x;
        const uint32_t dst = stage_base + r * 128 + ((chunk ^ (r & 7)) << 4);
        cp_async_16(dst, src, valid);
      }
      cp_async_commit();
      if (i >= kLag) {
        cp_async_wait<kLag>();
        fence_proxy_async_smem();
        mbar_arrive(&full[(i - kLag) % kStages]);
      }
    }
    cp_async_wait<0>();
    fence_proxy_async_smem();
    for (int i = max(0, nkb - kLag); i < nkb; ++i) mbar_arrive(&full[i % kStages]);
    }  // gather mode
    const int row = warp * 32 + lane;
    const int m = m0 + row;
    const bool row_ok = row < mvalid;
    const bool has_res = a.res != nullptr && row_ok;
    const __nv_bfloat16* res_row = has_res ? a.res + static_cast<size_t>(m) * a.cout + n0 : nullptr;
    // this thread's first residual chunk: in flight while the last loads land / MMAs drain
    uint4 res_cur[4];
    if (has_res && !RT) {
#pragma unroll
      for (int q = 0; q < 4; ++q) res_cur[q] = ldg_nc16(res_row + 8 * q);
    }
    if (ts && threadIdx.x == 0) ts[3] = gtimer();

    // ---------------- epilogue ----------------
    __syncwarp();
    mbar_wait(tmem_full, 0);
    tc_fence_after();
    if (threadIdx.x == 0) pdl_trigger();  // mainloop done: let the next layer start its prologue
    asm volatile("bar.sync 1, 128;" ::: "memory");  // scale/bias in smem visible to all producers
    if (ts && threadIdx.x == 0) ts[4] = gtimer();
    const uint32_t t_row = tmem_base + (static_cast<uint32_t>(warp * 32) << 16);
    if (BN == 64 && a.cluster_split) {
      // (cluster barrier and reduction below, executed by all 192 threads)
    } else if (a.splits == 1) {
      // Stage the bf16 tile in the (now idle) A ring as 64-column halves of
      // 128 B rows, 128B-swizzled (conflict-free 16 B writes, one row per
      // thread), then one TMA store per half: coalesced, asynchronous, and
      // rows past the image / tensor end are clipped by the tensor map.
      const uint32_t swz = static_cast<uint32_t>(row & 7);
      const int c1 = a.tma_a ? h0 * a.wo : m0;
      const int c2 = a.tma_a ? img : 0;
      if constexpr (RT) mbar_wait(res_bar, 0);
      // (the residual by chunk, the next chunk's loads in flight while this one is
      // packed: all of a row at once through cp.async into the idle B ring after
      // the accumulator is ready measured slower — layer1 conv3 9.1 -> 10.1 us at
      // batch 1, 76 -> 90 us at batch 64 — the first chunk here is in flight
      // during the mainloop already)
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 32) {
        uint32_t r[32];
        uint4 res_nxt[4];
        const uint32_t chunk0 = static_cast<uint32_t>((c0 & 63) >> 3);
        if constexpr (RT) {
          if (has_res) {  // this chunk of the row from the TMA-staged residual (same swizzle)
            const uint8_t* rp = (c0 < 64 ? res_half0 : res_half1) + row * 128;
#pragma unroll
            for (int q = 0; q < 4; ++q) res_cur[q] = *reinterpret_cast<const uint4*>(rp + (((chunk0 + q) ^ swz) << 4));
          }
        } else if (has_res && c0 + 32 < BN) {
#pragma unroll
          for (int q = 0; q < 4; ++q) res_nxt[q] = ldg_nc16(res_row + c0 + 32 + 8 * q);
        }
        tmem_ld_32x32b_x32(t_row + c0, r);
        uint8_t* rowp = out_half(c0 >> 6) + row * 128;
        uint4 pk[4];
        pack_row32(a, c0, reinterpret_cast<const float*>(r), s_scale, s_bias, res_cur, has_res, pk);
#pragma unroll
        for (int q = 0; q < 4; ++q) *reinterpret_cast<uint4*>(rowp + (((chunk0 + q) ^ swz) << 4)) = pk[q];
        if constexpr (!RT) {
#pragma unroll
          for (int q = 0; q < 4; ++q) res_cur[q] = res_nxt[q];
        }
      }
      fence_proxy_async_smem();  // generic-proxy smem writes -> visible to the TMA engine
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (threadIdx.x == 0) {
#pragma unroll
        for (int h = 0; h < BN / 64; ++h)
          tma_store_3d(&ymap, out_half(h), n0 + h * 64, c1, c2);
        bulk_commit();
        bulk_wait_read();
      }
    } else {
      // Split-K: every split reduces its fp32 partial into the zeroed tile
      // accumulator (red.add at L2), then takes a ticket; the split that
      // arrives last reads the sum, re-zeroes it, runs the epilogue and
      // re-arms the ticket for the next launch. Nobody waits for anybody.
      const int tile = tile_m * gridDim.y + tile_n;
      int* ticket_ctr = a.counters + 2 * tile;
      float* acc_row = a.ws + static_cast<size_t>(tile) * (kBM * BN) + static_cast<size_t>(row) * BN;
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 32) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(t_row + c0, r);
        if (row_ok) {
#pragma unroll
          for (int q = 0; q < 8; ++q)
            red_add_v4(acc_row + c0 + 4 * q, __uint_as_float(r[4 * q]), __uint_as_float(r[4 * q + 1]),
                       __uint_as_float(r[4 * q + 2]), __uint_as_float(r[4 * q + 3]));
        }
      }
      __threadfence();
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (threadIdx.x == 0) *last_flag = (atomicAdd(ticket_ctr, 1) == a.splits - 1);
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (*last_flag) {
        __threadfence();
        if (row_ok) {
#pragma unroll 1
          for (int c0 = 0; c0 < BN; c0 += 32) {
            float4* src = reinterpret_cast<float4*>(acc_row + c0);
            float4 part[8];
            uint4 res_nxt[4];
#pragma unroll
            for (int q = 0; q < 8; ++q) part[q] = __ldcg(src + q);  // all loads in flight together
            if (has_res && c0 + 32 < BN) {
#pragma unroll
              for (int q = 0; q < 4; ++q) res_nxt[q] = ldg_nc16(res_row + c0 + 32 + 8 * q);
            }
#pragma unroll
            for (int q = 0; q < 8; ++q) __stcg(src + q, make_float4(0.f, 0.f, 0.f, 0.f));  // re-arm
            finalize_row32(a, m, n0 + c0, c0, reinterpret_cast<const float*>(part), s_scale, s_bias,
                           res_cur, has_res);
#pragma unroll
            for (int q = 0; q < 4; ++q) res_cur[q] = res_nxt[q];
          }
        }
        if (threadIdx.x == 0) ticket_ctr[0] = 0;
      }
    }
  } else if (warp == 4) {
    // ---------------- weight producer (TMA) ----------------
    if (lane == 0 && !a.tma_a) {
      // weights are constant: stream them before waiting on the previous layer
      for (int i = 0; i < nkb; ++i) {
        const int s = i % kStages;
        if (i >= kStages) mbar_wait(&empty[s], ((i / kStages) & 1) ^ 1);
        mbar_arrive_expect_tx(&full[s], L::kBBytes);
        tma_load_2d(&wmap, &full[s], sB + s * L::kBBytes, (kb_begin + i) * kBK, n0);
      }
    } else if (lane == 0) {
      // TMA mode: activations too. K block kb = (kernel position r,s ; 64-channel
      // block c); its A tile is the 4-D box {64 ch, wo cols, th rows, 1 image}
      // at input (c, s - pad, h0*stride - pad + r, img), traversed with the conv
      // stride; padding comes from TMA's zero fill of out-of-bounds elements.
      const uint32_t a_bytes = static_cast<uint32_t>(a.th * a.wo * 128 * a.ipt);
      auto load_a = [&](int i, int s) {
        const int kb = kb_begin + i;
        if (a.stem_tma) {  // K block = kernel row kb: windows of th output rows at padded input row h0*s + kb
          tma_load_4d(&amap, &full[s], sA + s * L::kABytes, 0, 0, h0 * a.stride + kb, img);
          return;
        }
        if (kb >= a.kb_seg1) {  // DARIS_CONV_DUAL branch: 1x1 over x2, sampled with stride2
          tma_load_4d(&amap2, &full[s], sA + s * L::kABytes, (kb - a.kb_seg1) * kBK, 0, h0 * a.stride2, img);
          return;
        }
        const int kpos = fdiv(kb, a.d_cinb);
        const int cb = kb - kpos * a.cin_blocks;
        const int r_ = fdiv(kpos, a.d_kw), s_ = kpos - r_ * a.kw;
        tma_load_4d(&amap, &full[s], sA + s * L::kABytes, cb * kBK, s_ - a.pad, h0 * a.stride - a.pad + r_, img);
      };
      const int pre = min(nkb, kStages);
      for (int i = 0; i < pre; ++i) {  // weights first: they do not depend on the previous layer
        mbar_arrive_expect_tx(&full[i], L::kBBytes + a_bytes);
        tma_load_2d(&wmap, &full[i], sB + i * L::kBBytes, (kb_begin + i) * kBK, n0);
      }
      pdl_wait();
      auto load_res = [&]() {
        mbar_arrive_expect_tx(res_bar, static_cast<uint32_t>((BN / 64) * a.box_rows * 128 * a.ipt));
        tma_load_3d(&rmap, res_bar, res_half0, n0, h0 * a.wo, img);
        if (BN == 128) tma_load_3d(&rmap, res_bar, res_half1, n0 + 64, h0 * a.wo, img);
      };
      if constexpr (RT) {
        if (nkb < kStages) load_res();  // stage nkb is never used by the K loop
      }
      for (int i = 0; i < pre; ++i) load_a(i, i);
      for (int i = pre; i < nkb; ++i) {
        const int s = i % kStages;
        mbar_wait(&empty[s], ((i / kStages) & 1) ^ 1);
        mbar_arrive_expect_tx(&full[s], L::kBBytes + a_bytes);
        tma_load_2d(&wmap, &full[s], sB + s * L::kBBytes, (kb_begin + i) * kBK, n0);
        load_a(i, s);
      }
      if constexpr (RT) {
        if (nkb >= kStages) {  // as K block nkb would: once the MMAs have freed stage rs
          mbar_wait(&empty[rs], ((nkb / kStages) & 1) ^ 1);
          load_res();
        }
      }
    }
  } else {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      constexpr uint32_t idesc = umma_idesc_bf16(kBM, BN);
      const uint32_t sA_u32 = smem_u32(sA), sB_u32 = smem_u32(sB);
      for (int i = 0; i < nkb; ++i) {
        const int s = i % kStages;
        mbar_wait(&full[s], (i / kStages) & 1);
        tc_fence_after();
        const uint64_t bdesc = umma_desc_k_sw128(sB_u32 + s * L::kBBytes);
        const uint64_t adesc = umma_desc_k_sw128(sA_u32 + s * L::kABytes);
#pragma unroll
        for (int k = 0; k < kBK / 16; ++k) {
          // +32 B along K inside the 128 B swizzle atom = +2 in the encoded start address
          umma_bf16(tmem_base, adesc + 2 * k, bdesc + 2 * k, idesc, (i > 0 || k > 0) ? 1u : 0u);
        }
        umma_commit(&empty[s]);
      }
      umma_commit(tmem_full);
    }
  }

  if (BN == 64 && a.cluster_split) {
    // Split-K inside one cluster, pulled: every CTA stages its fp32 partial tile
    // in its own (now idle) A ring, row per thread, 16-B chunks XOR-swizzled by
    // row; after one cluster barrier CTA r reduces rows [r*V/S, (r+1)*V/S)
    // (V = the tile's valid rows) by reading them from every CTA's stage (ld.shared::cluster,
    // 8 lanes per 256-B row), applies the epilogue and stores. Staging + pulling
    // measured 1.44 us per exchange vs 2.08 us for st.async pushes of whole
    // rows (tools/dsmem_probe.cu, profiles/r02_dsmem_probe.txt).
    const int S = a.splits;
    float* stage = reinterpret_cast<float*>(sA);  // [128][BN] fp32
    __syncwarp();
    if (ts && threadIdx.x == 0) ts[8] = gtimer();
    if (warp < 4) {
      const int row = warp * 32 + lane;
      const uint32_t t_row = tmem_base + (static_cast<uint32_t>(warp * 32) << 16);
#pragma unroll
      for (int c0 = 0; c0 < BN; c0 += 32) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(t_row + c0, r);  // warp-collective: every lane loads
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int chunk = (c0 >> 2) + q;  // 16-B chunk index in the row (BN / 4 per row)
          *reinterpret_cast<float4*>(stage + row * BN + ((chunk ^ (row & 15)) << 2)) =
              make_float4(__uint_as_float(r[4 * q]), __uint_as_float(r[4 * q + 1]), __uint_as_float(r[4 * q + 2]),
                          __uint_as_float(r[4 * q + 3]));
        }
      }
    }
    cluster_sync();  // every split's partial is staged
    if (ts && threadIdx.x == 0) ts[9] = gtimer();
    {  // all six warps pull (the TMA and MMA warps are idle by now): more DSMEM loads in flight
      // the tile's valid rows split evenly over the S CTAs (layer4 at batch 1:
      // 49 rows -> 16 / 16 / 17, not 43 / 6 / 0)
      const int r_begin = (split * mvalid) / S, r_end = ((split + 1) * mvalid) / S;
      const int valid = r_end - r_begin;
      float* s_scale = reinterpret_cast<float*>(smem + L::kEpiOff);
      float* s_bias = s_scale + BN;
      const uint32_t stage_u32 = smem_u32(stage);
      const int items = valid * (BN / 8);  // (row, 8-column group)
      for (int it = threadIdx.x; it < items; it += kThreads) {
        const int j = it / (BN / 8), g = it % (BN / 8);
        const int rr = r_begin + j;
        const int m = m0 + rr;
        const int c = g * 8;
        const size_t off = static_cast<size_t>(m) * a.cout + n0 + c;
        uint4 rv = make_uint4(0, 0, 0, 0);
        if (a.res != nullptr) rv = ldg_nc16(a.res + off);
        const uint32_t a0 = stage_u32 + static_cast<uint32_t>((rr * BN + (((2 * g) ^ (rr & 15)) << 2)) * 4);
        const uint32_t a1 = stage_u32 + static_cast<uint32_t>((rr * BN + (((2 * g + 1) ^ (rr & 15)) << 2)) * 4);
        float v[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll 1
        for (int k0 = 0; k0 < S; k0 += 4) {  // S <= 8: up to 4 peers' chunks in flight at once
          float4 p0[4], p1[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            if (k0 + k < S) {
              p0[k] = ld_dsmem_f4(dsmem_map(a0, k0 + k));
              p1[k] = ld_dsmem_f4(dsmem_map(a1, k0 + k));
            }
          }
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            if (k0 + k < S) {
              v[0] += p0[k].x; v[1] += p0[k].y; v[2] += p0[k].z; v[3] += p0[k].w;
              v[4] += p1[k].x; v[5] += p1[k].y; v[6] += p1[k].z; v[7] += p1[k].w;
            }
          }
        }
        float rf[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        if (a.res != nullptr) {
          const uint32_t rr4[4] = {rv.x, rv.y, rv.z, rv.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 f = unpack_bf16x2(rr4[e]);
            rf[2 * e] = f.x;
            rf[2 * e + 1] = f.y;
          }
        }
        float o[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) o[e] = v[e] * s_scale[c + e] + s_bias[c + e] + rf[e];
        if (a.relu == 1) {
#pragma unroll
          for (int e = 0; e < 8; ++e) o[e] = fmaxf(o[e], 0.f);
        } else if (a.relu == 6) {
#pragma unroll
          for (int e = 0; e < 8; ++e) o[e] = fminf(fmaxf(o[e], 0.f), 6.f);
        }
        uint4 pk;
        pk.x = pack_bf16x2(o[0], o[1]);
        pk.y = pack_bf16x2(o[2], o[3]);
        pk.z = pack_bf16x2(o[4], o[5]);
        pk.w = pack_bf16x2(o[6], o[7]);
        *reinterpret_cast<uint4*>(a.y + off) = pk;
      }
    }
    if (ts && threadIdx.x == 0) ts[10] = gtimer();
    cluster_sync();  // nobody leaves (or reuses its stage) while a peer may still read it
    if (ts && threadIdx.x == 0) ts[11] = gtimer();
  }
  if (ts && threadIdx.x == 0) ts[5] = gtimer();
  tc_fence_before();
  __syncthreads();
  if (warp == 4) {
    tc_fence_after();
    tmem_dealloc<BN>(tmem_base);
  }
  if (ts && threadIdx.x == 0) ts[6] = gtimer();
}

// ---------------------------------------------------------------------------
// ---------------------------------------------------------------------------
// CTA-pair conv for large-M launches (batched jobs, single-tenant batching):
// a (2,1,1) cluster on one TPC runs one UMMA M = 256 tile with
// tcgen05.mma.cta_group::2. Each CTA loads its own 128-row activation tile (the
// same TMA boxes as above: th whole output rows, stem windows or the fused
// downsample branch) and HALF of the BN-wide weight tile, both into the same
// smem offsets; both CTAs' loads complete on the leader's full barrier
// (cta_group::2 TMA), the leader alone issues the MMAs, and its commits arrive
// on both CTAs' empty / accumulator barriers (multicast). Every CTA then runs
// the TMA-store epilogue of its own 128 accumulator rows from its own TMEM.
// Per SM and K block this moves 16 KB of A + BN/2 x 128 B of B for a
// 128 x BN x 64 MMA share — half the weight traffic of a one-CTA tile.

template <int BN, int ST>
struct PairLayout {
  static constexpr int kABytes = kBM * 128;
  static constexpr int kBBytes = (BN / 2) * 128;
  static constexpr int kAOff = 0;
  static constexpr int kBOff = ST * kABytes;
  static constexpr int kBarOff = kBOff + ST * kBBytes;
  static constexpr int kEpiOff = kBarOff + 256;
  static constexpr int kTotal = kEpiOff + 2 * BN * 4 + 1024;
  static_assert((BN / 64) * kBM * 128 <= ST * kABytes, "output staging must fit in the A ring");
};

template <int BN, int ST>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    conv_pair_kernel(const __grid_constant__ CUtensorMap wmap, const __grid_constant__ CUtensorMap amap,
                     const __grid_constant__ CUtensorMap ymap, const __grid_constant__ CUtensorMap amap2,
                     const __grid_constant__ CUtensorMap /*rmap: unused*/, const ConvArgs a) {
  using L = PairLayout<BN, ST>;
  extern __shared__ uint8_t smem_raw[];
  // 1024-B aligned by pointer arithmetic on smem_raw (an integer round trip would
  // lose the shared address space: every smem access would become a generic LD/ST)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem + L::kAOff;
  uint8_t* sB = smem + L::kBOff;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::kBarOff);
  uint64_t* empty = full + ST;
  uint64_t* tmem_full = empty + ST;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const int tile_m = blockIdx.x, tile_n = blockIdx.y;
  const int q_img = fdiv(tile_m, a.d_tiles_h);
  const int img = q_img * a.ipt;
  const int h0 = (tile_m - q_img * a.tiles_h) * a.th;
  const int m0 = img * (a.ho * a.wo) + h0 * a.wo;
  // an odd M-tile count leaves the last pair's second CTA a phantom tile past
  // the last image: its boxes read zeros and its stores are clipped
  const int mvalid = img < a.n ? min(a.th, a.ho - h0) * a.wo * min(a.ipt, a.n - img) : 0;
  const int n0 = tile_n * BN;
  const int nkb = a.num_kb;

  if (threadIdx.x == 0) {
    for (int s = 0; s < ST; ++s) {
      mbar_init(&full[s], 1);   // the leader's producer arms it for both CTAs' bytes
      mbar_init(&empty[s], 1);  // one multicast commit from the leader's MMA thread
    }
    mbar_init(tmem_full, 1);
    fence_barrier_init();
  }
  if (warp == 4) {
    if (lane == 0) DBG_IN(0);
    tmem_alloc_cg2<BN>(tmem_slot);
    if (lane == 0) DBG_OUT(0);
    if (lane == 0) {
      tma_prefetch_desc(&wmap);
      tma_prefetch_desc(&amap);
      tma_prefetch_desc(&ymap);
      if (a.kb_seg1 < a.num_kb) tma_prefetch_desc(&amap2);
    }
  }
  tc_fence_before();
  if (threadIdx.x == 0) DBG_IN(1);
  cluster_sync();  // both CTAs' barriers initialised and TMEM allocated before any cross-CTA traffic
  if (threadIdx.x == 0) DBG_OUT(1);
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp < 4) {
    float* s_scale = reinterpret_cast<float*>(smem + L::kEpiOff);
    float* s_bias = s_scale + BN;
    for (int c = threadIdx.x; c < BN; c += 128) {
      s_scale[c] = __ldg(a.scale + n0 + c);
      s_bias[c] = __ldg(a.bias + n0 + c);
    }
    pdl_wait();  // the residual comes from an earlier layer
    const int row = warp * 32 + lane;
    const bool row_ok = row < mvalid;
    const bool has_res = a.res != nullptr && row_ok;
    const __nv_bfloat16* res_row = has_res ? a.res + static_cast<size_t>(m0 + row) * a.cout + n0 : nullptr;
    uint4 res_cur[4];
    if (has_res) {
#pragma unroll
      for (int q = 0; q < 4; ++q) res_cur[q] = ldg_nc16(res_row + 8 * q);
    }
    __syncwarp();
    PAIR_WAIT(tmem_full, 0, 1);
    tc_fence_after();
    if (threadIdx.x == 0) pdl_trigger();
    asm volatile("bar.sync 1, 128;" ::: "memory");
    const uint32_t t_row = tmem_base + (static_cast<uint32_t>(warp * 32) << 16);
    uint8_t* stage = sA;
    const uint32_t swz = static_cast<uint32_t>(row & 7);
#pragma unroll 1
    for (int c0 = 0; c0 < BN; c0 += 32) {
      uint32_t r[32];
      uint4 res_nxt[4];
      if (has_res && c0 + 32 < BN) {
#pragma unroll
        for (int q = 0; q < 4; ++q) res_nxt[q] = ldg_nc16(res_row + c0 + 32 + 8 * q);
      }
      tmem_ld_32x32b_x32(t_row + c0, r);
      uint8_t* rowp = stage + (c0 >> 6) * (kBM * 128) + row * 128;
      const uint32_t chunk0 = static_cast<uint32_t>((c0 & 63) >> 3);
      uint4 pk[4];
      pack_row32(a, c0, reinterpret_cast<const float*>(r), s_scale, s_bias, res_cur, has_res, pk);
#pragma unroll
      for (int q = 0; q < 4; ++q) *reinterpret_cast<uint4*>(rowp + (((chunk0 + q) ^ swz) << 4)) = pk[q];
#pragma unroll
      for (int q = 0; q < 4; ++q) res_cur[q] = res_nxt[q];
    }
    fence_proxy_async_smem();
    asm volatile("bar.sync 1, 128;" ::: "memory");
    if (threadIdx.x == 0 && mvalid > 0) {
#pragma unroll
      for (int h = 0; h < BN / 64; ++h) tma_store_3d(&ymap, stage + h * (kBM * 128), n0 + h * 64, h0 * a.wo, img);
      bulk_commit();
      bulk_wait_read();
    }
  } else if (warp == 4) {
    if (lane == 0) {
      const uint32_t a_bytes = static_cast<uint32_t>(a.th * a.wo * 128 * a.ipt);
      const uint32_t stage_tx = 2u * (a_bytes + static_cast<uint32_t>(L::kBBytes));  // both CTAs
      const int nb0 = n0 + static_cast<int>(rank) * (BN / 2);
      auto load_a = [&](int kb, int s) {
        if (a.stem_tma) {
          tma_load_4d_cg2(&amap, &full[s], sA + s * L::kABytes, 0, 0, h0 * a.stride + kb, img);
          return;
        }
        if (kb >= a.kb_seg1) {
          tma_load_4d_cg2(&amap2, &full[s], sA + s * L::kABytes, (kb - a.kb_seg1) * kBK, 0, h0 * a.stride2, img);
          return;
        }
        const int kpos = fdiv(kb, a.d_cinb);
        const int cb = kb - kpos * a.cin_blocks;
        const int r_ = fdiv(kpos, a.d_kw), s_ = kpos - r_ * a.kw;
        tma_load_4d_cg2(&amap, &full[s], sA + s * L::kABytes, cb * kBK, s_ - a.pad, h0 * a.stride - a.pad + r_,
                        img);
      };
      const int pre = min(nkb, ST);
      for (int i = 0; i < pre; ++i) {  // weights first: they do not depend on the previous layer
        if (rank == 0) mbar_arrive_expect_tx(&full[i], stage_tx);
        tma_load_2d_cg2(&wmap, &full[i], sB + i * L::kBBytes, i * kBK, nb0);
      }
      DBG_IN(3);
      pdl_wait();
      DBG_OUT(3);
      for (int i = 0; i < pre; ++i) load_a(i, i);
      for (int i = pre; i < nkb; ++i) {
        const int s = i % ST;
        PAIR_WAIT(&empty[s], ((i / ST) & 1) ^ 1, 2);
        if (rank == 0) mbar_arrive_expect_tx(&full[s], stage_tx);
        tma_load_2d_cg2(&wmap, &full[s], sB + s * L::kBBytes, i * kBK, nb0);
        load_a(i, s);
      }
    }
  } else if (rank == 0 && lane == 0) {
    // ---------------- MMA issuer (leader only): D[256 x BN] over both CTAs ----------------
    constexpr uint32_t idesc = umma_idesc_bf16(2 * kBM, BN);
    const uint32_t sA_u32 = smem_u32(sA), sB_u32 = smem_u32(sB);
    for (int i = 0; i < nkb; ++i) {
      const int s = i % ST;
      PAIR_WAIT(&full[s], (i / ST) & 1, 3);
      tc_fence_after();
      const uint64_t adesc = umma_desc_k_sw128(sA_u32 + s * L::kABytes);
      const uint64_t bdesc = umma_desc_k_sw128(sB_u32 + s * L::kBBytes);
#pragma unroll
      for (int k = 0; k < kBK / 16; ++k)
        umma_bf16_cg2(tmem_base, adesc + 2 * k, bdesc + 2 * k, idesc, (i > 0 || k > 0) ? 1u : 0u);
      umma_commit_cg2(&empty[s], 0x3);
    }
    umma_commit_cg2(tmem_full, 0x3);
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) DBG_IN(2);
  cluster_sync();  // the peer's smem / TMEM are done with before either CTA frees TMEM or exits
  if (threadIdx.x == 0) DBG_OUT(2);
  if (warp == 4) {
    tc_fence_after();
    tmem_dealloc_cg2<BN>(tmem_base);
  }
}

// ------------------------------------------------------------------ host side
static PFN_cuTensorMapEncodeTiled_v12000 get_encode_fn() {
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

// Whole images per M tile: with one image per tile a map of <= 64 output pixels
// (ResNet layer4's 7x7 at batch > 1) leaves most of the 128-row tile idle; k =
// 128 / (ho*wo) images ride in one tile as the TMA boxes' image extent (the
// rows stay image-major, so A, residual and output boxes line up). Only when
// a tile already holds whole images (th == ho); stems excluded (their window
// boxes are per image row). DARIS_CONV_IMGS=0 keeps one image per tile (A/B).
static int imgs_per_tile(const daris_conv_desc* d, bool tma_a, int th) {
  static const bool off = [] {
    const char* e = std::getenv("DARIS_CONV_IMGS");
    return e && std::atoi(e) == 0;
  }();
  if (off || !tma_a || th < d->ho || d->cin == 8 || (d->flags & DARIS_CONV_PADDED_INPUT)) return 1;
  return std::max(1, std::min(kBM / (d->ho * d->wo), d->n));
}

template <int BN, int ST, bool PAIR, bool RT = false>
constexpr auto conv_kernel_fn() {
  if constexpr (PAIR) return conv_pair_kernel<BN, ST>;
  else return conv_igemm_tc_kernel<BN, ST, RT>;
}
template <int BN, int ST, bool PAIR>
constexpr int conv_smem_bytes() {
  if constexpr (PAIR) return PairLayout<BN, ST>::kTotal;
  else return SmemLayout<BN, ST>::kTotal;
}

template <int BN, int ST = Depth<BN>::kStages, bool PAIR = false>
static int launch_bn(const daris_conv_desc* d, const daris_conv_plan_t& pl, cudaStream_t st) {
  constexpr int kSmem = conv_smem_bytes<BN, ST, PAIR>();
  auto kernel = conv_kernel_fn<BN, ST, PAIR>();
  auto encode = get_encode_fn();
  if (!encode) return DARIS_K_NO_DRIVER;
  const int K = ((d->flags & DARIS_CONV_PADDED_INPUT) ? d->kh * 64 : d->kh * d->kw * d->cin) +
                ((d->flags & DARIS_CONV_DUAL) ? d->cin2 : 0);
  CUtensorMap map;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(d->cout)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(K) * 2};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(kBK), static_cast<cuuint32_t>(PAIR ? BN / 2 : BN)};  // a pair: half each
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(d->weight), dims, strides, box,
                      estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return DARIS_K_BAD_ARG;
  CUtensorMap amap;
  std::memset(&amap, 0, sizeof(amap));
  const bool stem_tma = pl.tma_rows > 0 && d->cin == 8;
  const int ipt = imgs_per_tile(d, pl.tma_rows > 0, pl.tma_rows);
  if (stem_tma) {
    // zero-bordered NHWC8 input [n][hp][wp][8]: dim0 = the 64-element (128 B) window of
    // kw pixels x 8 channels starting at padded column ow*stride, dim1 = output column
    // (windows overlap: global stride stride*16 B), dim2 = padded input row, dim3 = image
    const int th = pl.tma_rows;
    const cuuint64_t hp = static_cast<cuuint64_t>(d->h) + 2 * d->pad;
    const cuuint64_t wp = static_cast<cuuint64_t>(d->w) + 2 * d->pad + 8;
    cuuint64_t adims[4] = {64, static_cast<cuuint64_t>(d->wo), hp, static_cast<cuuint64_t>(d->n)};
    cuuint64_t astr[3] = {static_cast<cuuint64_t>(d->stride) * 16, wp * 16, hp * wp * 16};
    cuuint32_t abox[4] = {64, static_cast<cuuint32_t>(d->wo), static_cast<cuuint32_t>(th * d->stride), 1};
    cuuint32_t aestr[4] = {1, 1, static_cast<cuuint32_t>(d->stride), 1};
    r = encode(&amap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(d->x), adims, astr, abox, aestr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return DARIS_K_BAD_ARG;
  } else if (pl.tma_rows > 0) {
    // activations NHWC as a 4-D tensor (c, w, h, n); one box = th output rows x wo
    // output columns x 64 channels, traversed with the conv stride
    const int th = pl.tma_rows;
    cuuint64_t adims[4] = {static_cast<cuuint64_t>(d->cin), static_cast<cuuint64_t>(d->w),
                           static_cast<cuuint64_t>(d->h), static_cast<cuuint64_t>(d->n)};
    cuuint64_t astr[3] = {static_cast<cuuint64_t>(d->cin) * 2, static_cast<cuuint64_t>(d->w) * d->cin * 2,
                          static_cast<cuuint64_t>(d->h) * d->w * d->cin * 2};
    cuuint32_t abox[4] = {static_cast<cuuint32_t>(kBK), static_cast<cuuint32_t>(d->wo * d->stride),
                          static_cast<cuuint32_t>(th * d->stride), static_cast<cuuint32_t>(ipt)};
    cuuint32_t aestr[4] = {1, static_cast<cuuint32_t>(d->stride), static_cast<cuuint32_t>(d->stride), 1};
    r = encode(&amap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(d->x), adims, astr, abox, aestr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return DARIS_K_BAD_ARG;
  }

  // epilogue by TMA store (splits == 1): the output as a 3-D tensor {cout, rows, images}
  // whose box is one M tile (th whole output rows of one image, or 128 flat rows)
  const bool tma_c = pl.splits == 1;
  CUtensorMap ymap;
  std::memset(&ymap, 0, sizeof(ymap));
  int box_rows = 0;
  if (tma_c) {
    const bool per_image = pl.tma_rows > 0;
    const cuuint64_t rows = per_image ? static_cast<cuuint64_t>(d->ho) * d->wo
                                      : static_cast<cuuint64_t>(d->n) * d->ho * d->wo;
    cuuint64_t ydims[3] = {static_cast<cuuint64_t>(d->cout), rows, per_image ? static_cast<cuuint64_t>(d->n) : 1};
    cuuint64_t ystr[2] = {static_cast<cuuint64_t>(d->cout) * 2, rows * d->cout * 2};
    cuuint32_t ybox[3] = {64, static_cast<cuuint32_t>(per_image ? pl.tma_rows * d->wo : kBM),
                          static_cast<cuuint32_t>(per_image ? ipt : 1)};
    cuuint32_t yestr[3] = {1, 1, 1};
    r = encode(&ymap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, d->y, ydims, ystr, ybox, yestr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return DARIS_K_BAD_ARG;
    box_rows = static_cast<int>(ybox[1]);
  }

  const bool dual = (d->flags & DARIS_CONV_DUAL) != 0;
  CUtensorMap amap2;
  std::memset(&amap2, 0, sizeof(amap2));
  if (dual) {
    const int th = pl.tma_rows;
    cuuint64_t bdims[4] = {static_cast<cuuint64_t>(d->cin2), static_cast<cuuint64_t>(d->w2),
                           static_cast<cuuint64_t>(d->h2), static_cast<cuuint64_t>(d->n)};
    cuuint64_t bstr[3] = {static_cast<cuuint64_t>(d->cin2) * 2, static_cast<cuuint64_t>(d->w2) * d->cin2 * 2,
                          static_cast<cuuint64_t>(d->h2) * d->w2 * d->cin2 * 2};
    cuuint32_t bbox[4] = {static_cast<cuuint32_t>(kBK), static_cast<cuuint32_t>(d->wo * d->stride2),
                          static_cast<cuuint32_t>(th * d->stride2), static_cast<cuuint32_t>(ipt)};
    cuuint32_t bestr[4] = {1, static_cast<cuuint32_t>(d->stride2), static_cast<cuuint32_t>(d->stride2), 1};
    r = encode(&amap2, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(d->x2), bdims, bstr, bbox, bestr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return DARIS_K_BAD_ARG;
  }

  auto set_attrs = [&](auto fn) -> cudaError_t {
    set_max_carveout(reinterpret_cast<const void*>(fn));
    return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
  };
  static bool attr_set = false;  // per template instantiation
  if (!attr_set) {
    cudaError_t e = set_attrs(kernel);
    if (e != cudaSuccess) return e;
    if constexpr (!PAIR && BN <= 128) {
      e = set_attrs(conv_kernel_fn<BN, ST, false, true>());
      if (e != cudaSuccess) return e;
    }
    attr_set = true;
  }
  ConvArgs a;
  a.x = static_cast<const __nv_bfloat16*>(d->x);
  a.y = static_cast<__nv_bfloat16*>(d->y);
  a.res = static_cast<const __nv_bfloat16*>(d->residual);
  a.scale = d->scale;
  a.bias = d->bias;
  a.ws = d->workspace;
  a.counters = d->counters;
  a.n = d->n; a.h = d->h; a.w = d->w; a.cin = d->cin; a.cout = d->cout;
  a.kh = d->kh; a.kw = d->kw; a.stride = d->stride; a.pad = d->pad; a.ho = d->ho; a.wo = d->wo;
  a.M = d->n * d->ho * d->wo;
  a.relu = d->relu;
  a.cin_blocks = d->cin / kBK;
  a.d_howo = make_fdiv(d->ho * d->wo);
  a.d_wo = make_fdiv(d->wo);
  a.d_kw = make_fdiv(d->kw);
  a.d_cinb = make_fdiv(a.cin_blocks > 0 ? a.cin_blocks : 1);
  a.num_kb = stem_tma ? d->kh : d->cin == 8 ? (d->kh * d->kw + 7) / 8 : d->kh * d->kw * a.cin_blocks;
  a.kb_seg1 = a.num_kb;
  if (dual) a.num_kb += d->cin2 / kBK;
  a.stride2 = dual ? d->stride2 : 1;
  a.kb_per_split = pl.kb_per_split;
  a.splits = pl.splits;
  a.cluster_split = pl.cluster > 1 ? 1 : 0;
  a.tma_a = pl.tma_rows > 0 ? 1 : 0;
  a.tma_c = tma_c ? 1 : 0;
  a.stem_tma = stem_tma ? 1 : 0;
  a.box_rows = box_rows;
  a.th = pl.tma_rows > 0 ? pl.tma_rows : 1;
  a.ipt = ipt;
  a.tiles_h = (d->ho + a.th - 1) / a.th;
  a.d_tiles_h = make_fdiv(a.tiles_h);
  a.ts = reinterpret_cast<unsigned long long*>(d->timestamps);
  // the residual tile by TMA into a ring stage: one a short K loop never touches
  // (issued right after the dependency wait), else the first stage the MMAs free
  // after the last K block is loaded, so it lands during the mainloop instead of
  // being read chunk by chunk in the epilogue
  CUtensorMap rmap;
  std::memset(&rmap, 0, sizeof(rmap));
  a.res_tma = 0;
  if (!PAIR && tma_c && pl.tma_rows > 0 && d->residual && BN <= 128) {
    const cuuint64_t rows = static_cast<cuuint64_t>(d->ho) * d->wo;
    cuuint64_t rdims[3] = {static_cast<cuuint64_t>(d->cout), rows, static_cast<cuuint64_t>(d->n)};
    cuuint64_t rstr[2] = {static_cast<cuuint64_t>(d->cout) * 2, rows * d->cout * 2};
    cuuint32_t rbox[3] = {64, static_cast<cuuint32_t>(box_rows), static_cast<cuuint32_t>(ipt)};
    cuuint32_t restr[3] = {1, 1, 1};
    if (encode(&rmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(d->residual), rdims, rstr, rbox, restr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return DARIS_K_BAD_ARG;
    static const bool res_tma_off = std::getenv("DARIS_NO_RES_TMA") != nullptr;  // A/B knob
    a.res_tma = res_tma_off ? 0 : 1;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(PAIR ? (pl.tiles_m + 1) / 2 * 2 : pl.tiles_m, pl.tiles_n, pl.splits);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kSmem;
  cfg.stream = st;
  // experiment knob: without PDL a layer's CTAs are not launched early (an early
  // CTA holds smem/TMEM while it waits for its predecessor)
  static const bool no_pdl = std::getenv("DARIS_NO_PDL") != nullptr;
  cudaLaunchAttribute attr[2];
  cfg.attrs = attr;
  cfg.numAttrs = 0;
  if (!no_pdl) {
    attr[cfg.numAttrs].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[cfg.numAttrs].val.programmaticStreamSerializationAllowed = 1;
    cfg.numAttrs++;
  }
  if (!PAIR && pl.cluster > 1) {  // (the pair kernel's (2,1,1) cluster is compile-time)
    attr[cfg.numAttrs].id = cudaLaunchAttributeClusterDimension;
    attr[cfg.numAttrs].val.clusterDim.x = 1;
    attr[cfg.numAttrs].val.clusterDim.y = 1;
    attr[cfg.numAttrs].val.clusterDim.z = pl.cluster;
    cfg.numAttrs++;
  }
  if constexpr (!PAIR && BN <= 128) {
    if (a.res_tma)
      return static_cast<int>(
          cudaLaunchKernelEx(&cfg, conv_kernel_fn<BN, ST, false, true>(), map, amap, ymap, amap2, rmap, a));
  }
  return static_cast<int>(cudaLaunchKernelEx(&cfg, kernel, map, amap, ymap, amap2, rmap, a));
}


}  // namespace daris

extern "C" int daris_debug_pair_watch(void* host_mapped_words) {
#ifdef DARIS_PAIR_DEBUG
  void* dev = nullptr;
  if (host_mapped_words && cudaHostGetDevicePointer(&dev, host_mapped_words, 0) != cudaSuccess) return DARIS_K_BAD_ARG;
  cudaError_t e = cudaMemcpyToSymbol(daris::g_pair_watch, &dev, sizeof(dev));
  if (e == cudaSuccess) e = cudaMemcpyToSymbol(daris::g_wait_watch, &dev, sizeof(dev));
  return static_cast<int>(e);
#else
  (void)host_mapped_words;
  return DARIS_K_BAD_ARG;  // built without DARIS_PAIR_DEBUG
#endif
}

extern "C" int daris_device_sms(void) {
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

namespace daris {
// A 1x1 stride-1 unpadded convolution is a plain [M, cin] x [cin, cout] GEMM over
// the NHWC pixels, so its M tiles need not follow image rows: a TMA box of th
// whole output rows of one image leaves rows of the 128-row tile idle (7x7
// maps: 49 of 128; 14x14: 126 + 70), while the same tensor viewed as one image
// of M / w' rows of w' pixels, w' a divisor of M, tiles it almost exactly
// (ResNet-50 layer4 at batch 64: 64 -> 25 M tiles). Returns the descriptor to
// plan and launch: `tmp` with that view when it needs strictly fewer M tiles,
// else `d` (idempotent). DARIS_CONV_FLAT=0 keeps the per-image tiles (A/B).
static const daris_conv_desc* flat_view(const daris_conv_desc* d, daris_conv_desc* tmp) {
  static const bool off = [] {
    const char* e = std::getenv("DARIS_CONV_FLAT");
    return e && std::atoi(e) == 0;
  }();
  const bool dual = (d->flags & DARIS_CONV_DUAL) != 0;
  if (off || d->kh != 1 || d->kw != 1 || d->stride != 1 || d->pad != 0 || d->h != d->ho || d->w != d->wo ||
      d->cin % kBK != 0 || (d->flags & DARIS_CONV_PADDED_INPUT) || d->wo > kBM)
    return d;
  // the fused downsample (DUAL) samples x2 every stride2 pixels: images stack
  // along H only if output row r of the stack reads x2 row stride2 * r, i.e.
  // each image's x2 is exactly stride2 x the output, and the row width stays wo
  if (dual && (d->h2 != d->stride2 * d->ho || d->w2 != d->stride2 * d->wo)) return d;
  const int64_t M = static_cast<int64_t>(d->n) * d->ho * d->wo;
  const int th0 = std::max(1, std::min(d->ho, kBM / d->wo));
  const int64_t tiles0 = static_cast<int64_t>(d->n) * ((d->ho + th0 - 1) / th0);
  int64_t best = tiles0;
  int best_w = 0;
  for (int w = dual ? d->wo : kBM; w >= (dual ? d->wo : 1); --w) {
    if (M % w) continue;
    const int64_t rows = M / w, th = kBM / w;
    const int64_t tiles = (rows + th - 1) / th;
    if (tiles < best) best = tiles, best_w = w;
  }
  if (!best_w || M / best_w > (int64_t(1) << 30)) return d;
  // Only where it pays: per-image tiles that waste > 20 % of their rows, or a
  // grid of more than one wave of resident CTAs (3 per planned SM). A single
  // wave of 87.5 %-full tiles (batch-1 layer1: 28 -> 25 tiles) gets slightly
  // slower with fewer, fuller tiles (3.60 -> 3.62, 8.09 -> 8.29 us).
  const int budget = d->sm_budget > 0 ? d->sm_budget : daris_device_sms();
  const bool sparse = 5 * M < 4 * tiles0 * kBM;
  const bool waves = tiles0 * std::max(1, d->cout / 128) > 3 * budget;
  if (!sparse && !waves) return d;
  *tmp = *d;
  tmp->n = 1;
  tmp->h = tmp->ho = static_cast<int32_t>(M / best_w);
  tmp->w = tmp->wo = best_w;
  if (dual) tmp->h2 = d->n * d->h2;  // w2 = stride2 * wo unchanged
  return tmp;
}
}  // namespace daris

extern "C" int daris_conv_plan(const daris_conv_desc* d0, daris_conv_plan_t* out) {
  using namespace daris;
  if (!d0 || !out) return DARIS_K_BAD_ARG;
  daris_conv_desc flat;
  const daris_conv_desc* d = flat_view(d0, &flat);
  if ((d->cin % kBK != 0 && d->cin != 8) || d->cout % 64 != 0 || d->n < 1 || d->ho < 1 || d->wo < 1 ||
      d->kh < 1 || d->kw < 1 || d->stride < 1)
    return DARIS_K_BAD_SHAPE;
  const int M = d->n * d->ho * d->wo;
  const bool padded = (d->flags & DARIS_CONV_PADDED_INPUT) != 0;
  if (padded && (d->cin != 8 || d->kw > 8 || d->wo > kBM)) return DARIS_K_BAD_SHAPE;
  const bool dual = (d->flags & DARIS_CONV_DUAL) != 0;
  if (dual && (d->cin2 % kBK != 0 || d->cin2 <= 0 || d->stride2 < 1 || (d->ho - 1) * d->stride2 >= d->h2 ||
               (d->wo - 1) * d->stride2 >= d->w2 || d->cin % kBK != 0 || d->wo > kBM || d->residual))
    return DARIS_K_BAD_SHAPE;
  const int num_kb = (padded ? d->kh : d->cin == 8 ? (d->kh * d->kw + 7) / 8 : d->kh * d->kw * (d->cin / kBK)) +
                     (dual ? d->cin2 / kBK : 0);
  const int budget = d->sm_budget > 0 ? d->sm_budget : daris_device_sms();
  // Activations by TMA (4-D box of th whole output rows) unless the layer is a
  // stem (8 channels: pixel-chunk gather) or a box side would exceed 256.
  const int th = std::max(1, std::min(d->ho, kBM / d->wo));
  const bool tma_a = padded || dual ||
                     (d->cin % kBK == 0 && d->wo * d->stride <= 256 && th * d->stride <= 256 &&
                      d->wo <= kBM);
  const int tiles_h = (d->ho + th - 1) / th;
  const int ipt = imgs_per_tile(d, tma_a, th);
  const int tiles_m = !tma_a ? (M + kBM - 1) / kBM : ipt > 1 ? (d->n + ipt - 1) / ipt : d->n * tiles_h;
  int bn = d->block_n;
  if (bn == 0) {
    bn = d->cout % 128 == 0 ? 128 : 64;
    // 64-wide tiles when the 128-wide grid leaves resident CTA slots of the
    // planned SMs idle (3 per SM) and the 64-wide grid still fits in them:
    // twice the CTAs, each with half the epilogue, finish sooner. Batch 1 at 23
    // planned SMs: loaded capacity 15.2k -> 15.6k inf/s at 4x2, 21.5k -> 22.7k at
    // 16 jobs; large batches keep their 128-wide plans (profiles/r01_bn_rule_ab.txt).
    const int t128 = tiles_m * (d->cout / 128), t64 = 2 * t128;
    if (bn == 128 && t128 < 3 * budget && t64 <= 3 * budget)
      bn = 64;
  }
  if (bn != 64 && bn != 128 && bn != 256) return DARIS_K_BAD_SHAPE;
  if (d->cout % bn != 0) return DARIS_K_BAD_SHAPE;
  const int tiles_n = d->cout / bn;
  const int tiles = tiles_m * tiles_n;
  int splits = d->splits;
  if (splits <= 0) {
    // split-K costs one fix-up round trip (~2 us): only worth it for long K
    // loops on grids that leave most of the partition idle
    splits = 1;
    // (two or three split CTAs per planned SM: isolated job 0.343 -> 0.316 ms, but
    // loaded 4x2 capacity 17.7k -> 17.7k / 16.7k inf/s: profiles/r02_split_factor_ab.txt)
    if (tiles * 2 <= budget && num_kb >= 8) {
      splits = budget / tiles;
      const int max_by_k = num_kb / 4;  // keep >= 4 K blocks per split
      if (splits > max_by_k) splits = max_by_k;
      if (splits > 32) splits = 32;
      if (splits < 1) splits = 1;
    }
  }
  // a cluster holds at most 8 CTAs (portable size)
  if ((d->flags & DARIS_CONV_CLUSTER_SPLITK) && bn == 64 && splits > 8) splits = 8;
  if (splits > num_kb) splits = num_kb;
  int kbps = (num_kb + splits - 1) / splits;
  splits = (num_kb + kbps - 1) / kbps;  // no empty splits
  out->block_n = bn;
  out->splits = splits;
  out->kb_per_split = kbps;
  out->tiles_m = tiles_m;
  out->tiles_n = tiles_n;
  out->workspace_floats = splits > 1 ? static_cast<int64_t>(tiles) * kBM * bn : 0;  // zero-initialised
  out->counters = splits > 1 ? 2 * tiles : 0;  // ticket + done per tile
  out->ctas = tiles_m * tiles_n * splits;
  out->cluster = (splits > 1 && bn == 64 && (d->flags & DARIS_CONV_CLUSTER_SPLITK)) ? splits : 1;
  out->tma_rows = tma_a ? th : 0;
  // CTA pairs for large-M launches: TMA activations, no split-K, 128-wide (or
  // wider) tiles, at least one wave of tiles over the planned SMs, a K loop of
  // >= 16 blocks and <= 512 output channels. ResNet-50 at batch 64 on 148 SMs
  // (profiles/r02_pair_ab_b64.txt): 3x3 convs 24.2 -> 17.7 us (610 -> 835
  // TF/s), layer3 conv1 15.4 -> 11.7 us; the short-K / 1024-2048-channel
  // conv3s are faster as one-CTA tiles at 3 CTAs per SM (28.1 vs 32.8 us), and
  // after the epilogue diet so are the memory-bound 1x1 convs with long K
  // (layer4.0 conv1 18.6 -> 14.3 us, layer3 conv1 equal): pairs for spatial
  // kernels only (profiles/r02_pair_rule_1x1_ab.txt).
  // DARIS_CONV_PAIR=0 turns pairs off (A/B), =2 takes them wherever legal.
  static const int pair_mode = [] {
    const char* e = std::getenv("DARIS_CONV_PAIR");
    return e ? std::atoi(e) : 1;
  }();
  out->pair = 0;
  if (pair_mode > 0 && !(d->flags & DARIS_CONV_NO_PAIR) && tma_a && !padded && splits == 1 && (bn >= 128 || pair_mode == 2) &&
      tiles_m >= 2 &&
      (pair_mode == 2 || (tiles >= budget && num_kb >= 16 && d->cout <= 512 && d->kh * d->kw > 1)))
    out->pair = 1;
  if (out->cluster > 1) {  // partials reduce through DSMEM: no global scratch
    out->workspace_floats = 0;
    out->counters = 0;
  }
  return DARIS_K_OK;
}

extern "C" int daris_conv2d(const daris_conv_desc* d0, void* stream) {
  using namespace daris;
  if (!d0) return DARIS_K_BAD_ARG;
  daris_conv_desc flat;
  const daris_conv_desc* d = flat_view(d0, &flat);
  daris_conv_plan_t pl;
  int rc = daris_conv_plan(d, &pl);
  if (rc != DARIS_K_OK) return rc;
  if (!d->x || !d->y || !d->weight || !d->scale || !d->bias) return DARIS_K_BAD_ARG;
  if ((d->flags & DARIS_CONV_DUAL) && !d->x2) return DARIS_K_BAD_ARG;
  if (pl.splits > 1 && pl.cluster == 1 && (!d->workspace || !d->counters)) return DARIS_K_WORKSPACE;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (pl.pair) {
    switch (pl.block_n) {
      case 64: return launch_bn<64, 4, true>(d, pl, st);
      case 128: return launch_bn<128, 4, true>(d, pl, st);
      case 256: return launch_bn<256, 4, true>(d, pl, st);
    }
    return DARIS_K_BAD_SHAPE;
  }
  switch (pl.block_n) {
    case 64: return launch_bn<64>(d, pl, st);
    case 128: return launch_bn<128>(d, pl, st);
    case 256: return launch_bn<256>(d, pl, st);
  }
  return DARIS_K_BAD_SHAPE;
}
