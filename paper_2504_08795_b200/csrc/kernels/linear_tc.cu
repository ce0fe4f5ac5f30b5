// Linear layers on the sm_100a tensor cores (tcgen05 + TMEM + TMA), swap-AB:
//
//   D[o, b] = sum_k W[o, k] * X[b, k]     (UMMA M = 128 output features,
//                                           N = NB batch rows, K = 64 per stage)
//
// The weight matrix is the 128-row A operand and the (small) batch is the N
// side, so batch 1 wastes nothing but MMA slots — at batch <= 16 the layer is a
// weight stream and the tensor pipe is idle most of the time anyway, while at
// batch 64 (single-tenant batching) the same kernel is a real GEMM. Both
// operands arrive by TMA (2-D boxes, 128B swizzle; rows past `o` / `batch` are
// zero-filled by the tensor map), the weights before griddepcontrol.wait (they
// do not depend on the previous layer).
//
//   warps 0-3  epilogue: TMEM lane r = output feature o0 + r, one column per
//              batch row -> + bias -> act -> y[b][o] (a warp stores 128
//              contiguous bytes per batch row)
//   warp 4     TMA producer (one thread), TMEM owner
//   warp 5     MMA issuer (one thread)
//
// Split-K (weight-streaming shapes: few 128-row tiles, long K): every split
// adds its fp32 partial into a zeroed per-tile accumulator laid out
// [batch row][feature] (a warp's red.global.add covers one 128-B line), takes
// a ticket, and the last split runs the epilogue and re-zeroes accumulator and
// ticket for the next launch — the same protocol as the conv kernel's
// non-cluster split-K.
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <algorithm>
#include <cstring>
#include <mutex>
#include "sm100.cuh"
#include "../../../include/daris_kernels.h"

namespace daris {

constexpr int kLM = 128;      // output features per tile (UMMA M)
constexpr int kLK = 64;       // K per stage: 64 bf16 = one 128-B swizzle row
constexpr int kLThreads = 192;

template <int NB>
struct LinDepth {  // ring depth: ~100-150 KB of weights in flight per CTA
  static constexpr int kStages = NB <= 32 ? 6 : NB <= 64 ? 5 : NB <= 128 ? 4 : 3;
};

template <int NB, int ST>
struct LinLayout {
  static constexpr int kABytes = kLM * 128;
  static constexpr int kBBytes = NB * 128;
  static constexpr int kAOff = 0;
  static constexpr int kBOff = ST * kABytes;
  static constexpr int kBarOff = kBOff + ST * kBBytes;
  static constexpr int kTotal = kBarOff + 256 + 1024;  // + alignment slack
  static constexpr uint32_t kTmemCols = NB < 32 ? 32 : NB;
};

struct LinArgs {
  const float* bias;
  void* y;
  float* ws;
  int* counters;
  int batch, k, o, relu, y_bf16;
  int num_kb, kb_per_split, splits;
};

__device__ __forceinline__ void red_add_f32(float* p, float v) {
  asm volatile("red.global.add.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}

__device__ __forceinline__ void lin_store(const LinArgs& a, int b, int o, float v, float bias) {
  v += bias;
  if (a.relu == 1) v = fmaxf(v, 0.f);
  const size_t i = static_cast<size_t>(b) * a.o + o;
  if (a.y_bf16)
    static_cast<__nv_bfloat16*>(a.y)[i] = __float2bfloat16_rn(v);
  else
    static_cast<float*>(a.y)[i] = v;
}

template <int NB, int ST>
__global__ void __launch_bounds__(kLThreads, 1)
    linear_tc_kernel(const __grid_constant__ CUtensorMap wmap, const __grid_constant__ CUtensorMap xmap,
                     const LinArgs a) {
  using L = LinLayout<NB, ST>;
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
  int* last_flag = reinterpret_cast<int*>(tmem_slot + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int o0 = blockIdx.x * kLM;
  const int b0 = blockIdx.y * NB;
  const int kb_begin = blockIdx.z * a.kb_per_split;
  const int nkb = min(a.num_kb, kb_begin + a.kb_per_split) - kb_begin;

  if (threadIdx.x == 0) {
    for (int s = 0; s < ST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tmem_full, 1);
    fence_barrier_init();
  }
  if (warp == 4) {
    tmem_alloc<L::kTmemCols>(tmem_slot);
    if (lane == 0) {
      tma_prefetch_desc(&wmap);
      tma_prefetch_desc(&xmap);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 4) {
    if (lane == 0) {
      constexpr uint32_t kStageTx = L::kABytes + L::kBBytes;
      const int pre = min(nkb, ST);
      for (int i = 0; i < pre; ++i) {  // weights first: independent of the previous layer
        mbar_arrive_expect_tx(&full[i], kStageTx);
        tma_load_2d(&wmap, &full[i], sA + i * L::kABytes, (kb_begin + i) * kLK, o0);
      }
      pdl_wait();
      for (int i = 0; i < pre; ++i) tma_load_2d(&xmap, &full[i], sB + i * L::kBBytes, (kb_begin + i) * kLK, b0);
      for (int i = pre; i < nkb; ++i) {
        const int s = i % ST;
        mbar_wait(&empty[s], ((i / ST) & 1) ^ 1);
        mbar_arrive_expect_tx(&full[s], kStageTx);
        tma_load_2d(&wmap, &full[s], sA + s * L::kABytes, (kb_begin + i) * kLK, o0);
        tma_load_2d(&xmap, &full[s], sB + s * L::kBBytes, (kb_begin + i) * kLK, b0);
      }
    }
  } else if (warp == 5) {
    if (lane == 0) {
      constexpr uint32_t idesc = umma_idesc_bf16(kLM, NB);
      const uint32_t sA_u32 = smem_u32(sA), sB_u32 = smem_u32(sB);
      for (int i = 0; i < nkb; ++i) {
        const int s = i % ST;
        mbar_wait(&full[s], (i / ST) & 1);
        tc_fence_after();
        const uint64_t adesc = umma_desc_k_sw128(sA_u32 + s * L::kABytes);
        const uint64_t bdesc = umma_desc_k_sw128(sB_u32 + s * L::kBBytes);
#pragma unroll
        for (int k = 0; k < kLK / 16; ++k)
          umma_bf16(tmem_base, adesc + 2 * k, bdesc + 2 * k, idesc, (i > 0 || k > 0) ? 1u : 0u);
        umma_commit(&empty[s]);
      }
      umma_commit(tmem_full);
    }
  } else {
    // ---------------- epilogue ----------------
    const int row = warp * 32 + lane;
    const int orow = o0 + row;
    const bool row_ok = orow < a.o;
    const int nb_valid = min(NB, a.batch - b0);
    const float bias_o = (a.bias && row_ok) ? __ldg(a.bias + orow) : 0.f;  // before the wait: a constant
    mbar_wait(tmem_full, 0);
    tc_fence_after();
    if (threadIdx.x == 0) pdl_trigger();
    const uint32_t t_row = tmem_base + (static_cast<uint32_t>(warp * 32) << 16);
    constexpr int kChunk = NB < 32 ? NB : 32;
    if (a.splits == 1) {
#pragma unroll 1
      for (int c0 = 0; c0 < NB; c0 += kChunk) {
        uint32_t r[kChunk];
        tmem_ld_32x32b<kChunk>(t_row + c0, r);
        if (row_ok) {
#pragma unroll
          for (int j = 0; j < kChunk; ++j)
            if (c0 + j < nb_valid) lin_store(a, b0 + c0 + j, orow, __uint_as_float(r[j]), bias_o);
        }
      }
    } else {
      const int tile = blockIdx.x * gridDim.y + blockIdx.y;
      int* ticket = a.counters + tile;
      float* acc = a.ws + static_cast<size_t>(tile) * (NB * kLM);  // [NB][128]
#pragma unroll 1
      for (int c0 = 0; c0 < NB; c0 += kChunk) {
        uint32_t r[kChunk];
        tmem_ld_32x32b<kChunk>(t_row + c0, r);
        if (row_ok) {
#pragma unroll
          for (int j = 0; j < kChunk; ++j)
            if (c0 + j < nb_valid) red_add_f32(acc + (c0 + j) * kLM + row, __uint_as_float(r[j]));
        }
      }
      __threadfence();
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (threadIdx.x == 0) *last_flag = (atomicAdd(ticket, 1) == a.splits - 1);
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (*last_flag) {
        __threadfence();
        if (row_ok) {
          // a chunk of sums loaded together (one L2 round trip, not one per
          // batch row: the re-arming stores would otherwise order every load
          // behind the previous row's store), then re-armed and stored
#pragma unroll 1
          for (int c0 = 0; c0 < nb_valid; c0 += kChunk) {
            float v[kChunk];
#pragma unroll
            for (int j = 0; j < kChunk; ++j) v[j] = c0 + j < nb_valid ? __ldcg(acc + (c0 + j) * kLM + row) : 0.f;
#pragma unroll
            for (int j = 0; j < kChunk; ++j)
              if (c0 + j < nb_valid) __stcg(acc + (c0 + j) * kLM + row, 0.f);  // re-arm for the next launch
#pragma unroll
            for (int j = 0; j < kChunk; ++j)
              if (c0 + j < nb_valid) lin_store(a, b0 + c0 + j, orow, v[j], bias_o);
          }
        }
        if (threadIdx.x == 0) *ticket = 0;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 4) {
    tc_fence_after();
    tmem_dealloc<L::kTmemCols>(tmem_base);
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 lin_encode_fn() {
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

template <int NB, int ST = LinDepth<NB>::kStages>
static int launch_linear(const daris_linear_desc* d, const daris_linear_plan_t& pl, cudaStream_t st) {
  using L = LinLayout<NB, ST>;
  auto encode = lin_encode_fn();
  if (!encode) return DARIS_K_NO_DRIVER;
  CUtensorMap wmap, xmap;
  cuuint64_t wdims[2] = {static_cast<cuuint64_t>(d->k), static_cast<cuuint64_t>(d->o)};
  cuuint64_t wstr[1] = {static_cast<cuuint64_t>(d->k) * 2};
  cuuint32_t wbox[2] = {static_cast<cuuint32_t>(kLK), static_cast<cuuint32_t>(kLM)};
  cuuint32_t estr[2] = {1, 1};
  if (encode(&wmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(d->w), wdims, wstr, wbox, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return DARIS_K_BAD_ARG;
  cuuint64_t xdims[2] = {static_cast<cuuint64_t>(d->k), static_cast<cuuint64_t>(d->batch)};
  cuuint64_t xstr[1] = {static_cast<cuuint64_t>(d->k) * 2};
  cuuint32_t xbox[2] = {static_cast<cuuint32_t>(kLK), static_cast<cuuint32_t>(NB)};
  if (encode(&xmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(d->x), xdims, xstr, xbox, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return DARIS_K_BAD_ARG;
  static bool attr_set = false;  // per instantiation
  if (!attr_set) {
    set_max_carveout(reinterpret_cast<const void*>(linear_tc_kernel<NB, ST>));
    cudaError_t e =
        cudaFuncSetAttribute(linear_tc_kernel<NB, ST>, cudaFuncAttributeMaxDynamicSharedMemorySize, L::kTotal);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  LinArgs a;
  a.bias = d->bias;
  a.y = d->y;
  a.ws = d->workspace;
  a.counters = d->counters;
  a.batch = d->batch;
  a.k = d->k;
  a.o = d->o;
  a.relu = d->relu;
  a.y_bf16 = d->y_bf16;
  a.num_kb = d->k / kLK;
  a.kb_per_split = pl.kb_per_split;
  a.splits = pl.splits;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(pl.tiles_m, pl.tiles_n, pl.splits);
  cfg.blockDim = dim3(kLThreads);
  cfg.dynamicSmemBytes = L::kTotal;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return static_cast<int>(cudaLaunchKernelEx(&cfg, linear_tc_kernel<NB, ST>, wmap, xmap, a));
}

}  // namespace daris

extern "C" int daris_linear_plan(const daris_linear_desc* d, daris_linear_plan_t* out) {
  using namespace daris;
  if (!d || !out) return DARIS_K_BAD_ARG;
  if (d->batch < 1 || d->o < 1 || d->k < kLK || d->k % kLK != 0) return DARIS_K_BAD_SHAPE;
  const int nb = d->batch <= 16 ? 16 : d->batch <= 32 ? 32 : d->batch <= 64 ? 64 : d->batch <= 128 ? 128 : 256;
  const int tiles_m = (d->o + kLM - 1) / kLM;
  const int tiles_n = (d->batch + nb - 1) / nb;
  const int tiles = tiles_m * tiles_n;
  const int num_kb = d->k / kLK;
  const int budget = d->sm_budget > 0 ? d->sm_budget : daris_device_sms();
  int splits = d->splits;
  if (splits <= 0) {
    // about three CTAs per planned SM (weight streaming wants bytes in flight
    // on every SM), but at least max(2, NB / 8) K blocks per split: the fp32
    // reduction traffic grows with splits x NB (ResNet-50 head at batch 64:
    // 16 splits of 2 K blocks took 28.9 us, the atomics dominating)
    const int min_kb = std::max(2, nb / 8);
    splits = (3 * budget + tiles - 1) / tiles;
    splits = std::min(splits, std::max(1, num_kb / min_kb));
    splits = std::max(1, std::min(splits, 64));
  }
  if (splits > num_kb) splits = num_kb;
  const int kbps = (num_kb + splits - 1) / splits;
  splits = (num_kb + kbps - 1) / kbps;  // no empty splits
  out->block_n = nb;
  out->splits = splits;
  out->kb_per_split = kbps;
  out->tiles_m = tiles_m;
  out->tiles_n = tiles_n;
  out->workspace_floats = splits > 1 ? static_cast<int64_t>(tiles) * nb * kLM : 0;
  out->counters = splits > 1 ? tiles : 0;
  out->ctas = tiles * splits;
  return DARIS_K_OK;
}

extern "C" int daris_linear_tc(const daris_linear_desc* d, void* stream) {
  using namespace daris;
  daris_linear_plan_t pl;
  const int rc = daris_linear_plan(d, &pl);
  if (rc != DARIS_K_OK) return rc;
  if (!d->x || !d->w || !d->y) return DARIS_K_BAD_ARG;
  if (pl.splits > 1 && (!d->workspace || !d->counters)) return DARIS_K_WORKSPACE;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  switch (pl.block_n) {
    case 16: return launch_linear<16>(d, pl, st);
    case 32: return launch_linear<32>(d, pl, st);
    case 64: return launch_linear<64>(d, pl, st);
    case 128: return launch_linear<128>(d, pl, st);
    case 256: return launch_linear<256>(d, pl, st);
  }
  return DARIS_K_BAD_SHAPE;
}
