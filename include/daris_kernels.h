/* Stage-body kernels for DARIS on B200 (sm_100a) — C ABI.
 *
 * The reference (stagesim) has no tensor code: a stage is an opaque work
 * quantum `StageProfile(nominal_time, width)` (/root/reference/pkg/src/stagesim/model.py:24-27)
 * whose execution is the rate model `allocate_rates/next_completion/advance_progress`
 * (/root/reference/pkg/src/stagesim/gpu.py:167-240).  These entry points are
 * what replaces that rate model on real hardware: each DNN stage is a short
 * sequence of these launches, captured into one CUDA graph per (task, stage,
 * partition) by the executor (daris_exec.h).
 *
 * Layout conventions (all device pointers):
 *   activations  NHWC bf16, contiguous
 *   conv weights [Cout][KH][KW][Cin] bf16 (K-major rows for the tensor cores)
 *   folded BN    per-Cout fp32 scale and bias  (y = conv(x)*scale + bias)
 * All functions return 0 on success, a negative daris_kstatus on bad
 * arguments, or a positive cudaError_t from the launch.
 */
#ifndef DARIS_KERNELS_H
#define DARIS_KERNELS_H
#include <stddef.h>
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

enum daris_kstatus {
  DARIS_K_OK = 0,
  DARIS_K_BAD_SHAPE = -1,   /* a dimension the kernel cannot tile */
  DARIS_K_BAD_ARG = -2,     /* null pointer / misaligned buffer */
  DARIS_K_NO_DRIVER = -3,   /* cuTensorMapEncodeTiled unavailable */
  DARIS_K_WORKSPACE = -4    /* split-K scratch too small */
};

/* Implicit-GEMM convolution on tcgen05 (TMEM accumulators, TMA-fed weights,
 * cp.async-gathered activations) with a fused epilogue:
 *   y = act(conv(x, w) * scale + bias [+ residual])
 * Requirements: cin % 64 == 0 (or cin == 8: stem mode, NHWC8 input, K = kh*kw*8
 * zero-padded by TMA to a multiple of 64), cout % 64 == 0.
 * Split-K is used when the output tile count is small against `sm_budget`
 * (the SM count of the partition the stage runs in). */
typedef struct daris_conv_desc {
  const void* x;          /* [n][h][w][cin] bf16 */
  void* y;                /* [n][ho][wo][cout] bf16 */
  const void* residual;   /* like y, or NULL */
  const void* weight;     /* [cout][kh][kw][cin] bf16 */
  const float* scale;     /* [cout] */
  const float* bias;      /* [cout] */
  float* workspace;       /* split-K partials, daris_conv_plan() floats */
  int32_t* counters;      /* split-K tile counters, zero-initialised, self-resetting */
  int32_t n, h, w, cin, cout, kh, kw, stride, pad, ho, wo;
  int32_t relu;           /* 1: ReLU, 6: ReLU6, 0: none */
  int32_t block_n;        /* 0 = auto, else 64/128/256 */
  int32_t splits;         /* 0 = auto, else forced split-K factor */
  int32_t sm_budget;      /* SMs available to this launch (0 = whole device) */
  int32_t flags;          /* DARIS_CONV_CLUSTER_SPLITK: the launch context can co-schedule
                             clusters of up to 8 CTAs, so split-K partials are reduced through
                             distributed shared memory instead of global atomics */
  void* timestamps;       /* optional: 16 uint64 globaltimer stamps per CTA (profiling), or NULL */
  /* DARIS_CONV_DUAL: a second 1x1 convolution (a ResNet downsample branch) summed
   * into the same accumulator as extra K blocks: y = act(conv(x)*scale + x2_s*W2 + bias)
   * with x2_s = x2 sampled every stride2 pixels; weight is [cout][kh*kw*cin + cin2] */
  const void* x2;         /* [n][h2][w2][cin2] bf16, or NULL */
  int32_t h2, w2, cin2, stride2;
} daris_conv_desc;

enum {
  DARIS_CONV_CLUSTER_SPLITK = 1,
  /* 8-channel stems by TMA: x is stored zero-bordered as [n][h + 2*pad][w + 2*pad + 8][8]
   * and weight is [cout][kh][8][8] (the kw kernel columns padded to 8 pixel slots with
   * zeros): one K block = one kernel row, whose A tile is a single TMA box of
   * overlapping 128-B windows (requires cin == 8, kw <= 8, wo <= 128) */
  DARIS_CONV_PADDED_INPUT = 2,
  /* see x2 above: the primary conv must take the TMA path (cin % 64 == 0, wo <= 128);
   * the branch is 1x1, pad 0, (ho-1)*stride2 < h2, cin2 % 64 == 0 */
  DARIS_CONV_DUAL = 4,
  /* never plan CTA pairs for this launch (the executor's concurrent tenants) */
  DARIS_CONV_NO_PAIR = 8
};

typedef struct daris_conv_plan_t {
  int32_t block_n, splits, kb_per_split, tiles_m, tiles_n;
  int64_t workspace_floats; /* needed in desc.workspace */
  int32_t counters;         /* needed in desc.counters */
  int32_t ctas;
  int32_t cluster;          /* CTAs per cluster (split-K through DSMEM), 1 = none */
  int32_t tma_rows;         /* > 0: activations arrive by TMA, M tile = tma_rows whole output rows */
  int32_t pair;             /* 1: CTA pairs (cta_group::2, UMMA M = 256 over two M tiles, each CTA
                               loading half the weight tile) — large-M launches without split-K */
} daris_conv_plan_t;

int daris_conv_plan(const daris_conv_desc* d, daris_conv_plan_t* out);
int daris_conv2d(const daris_conv_desc* d, void* stream);

/* ResNet/VGG stem input pack: x fp32 NCHW [n][c][h][w] -> im2col rows
 * [n*ho*wo][kpad] bf16 with k = ci*kh*kw + r*kw + s (torch weight order),
 * zero-padded to kpad (a multiple of 64). Turns the c=3 stem into a GEMM. */
int daris_stem_im2col(const float* x, void* out, int32_t n, int32_t c, int32_t h, int32_t w, int32_t kh,
                      int32_t kw, int32_t stride, int32_t pad, int32_t ho, int32_t wo, int32_t kpad, void* stream);

/* NCHW fp32 -> NHWC bf16 with channels zero-padded to cpad (multiple of 8). */
/* NCHW fp32 -> NHWC bf16 (cpad channels) into the interior of a zero-bordered
 * [n][h + 2*border][w + 2*border + extra][cpad] buffer; the borders are never
 * written (allocate the buffer zeroed). Feeds DARIS_CONV_PADDED_INPUT stems. */
int daris_pack_nhwc_bordered(const float* x, void* out, int32_t n, int32_t c, int32_t h, int32_t w, int32_t cpad,
                             int32_t border, int32_t extra, void* stream);
int daris_pack_nhwc(const float* x, void* out, int32_t n, int32_t c, int32_t h, int32_t w, int32_t cpad,
                    void* stream);

/* Max pooling, NHWC bf16, c % 8 == 0. */
int daris_maxpool(const void* x, void* y, int32_t n, int32_t h, int32_t w, int32_t c, int32_t k, int32_t stride,
                  int32_t pad, int32_t ho, int32_t wo, void* stream);

/* Global average pooling NHWC bf16 [n][hw][c] -> fp32 [n][c]. */
int daris_avgpool(const void* x, float* y, int32_t n, int32_t hw, int32_t c, void* stream);

/* Linear layer for small batches (weight-streaming GEMV, HBM bound):
 * y[b][o] = act(sum_k x[b][k] * w[o][k] + bias[o]); x fp32 or bf16 (x_bf16=1),
 * y fp32 (y_bf16=0) or bf16. k % 8 == 0. */
int daris_linear(const void* x, int32_t x_bf16, const void* w, const float* bias, void* y, int32_t y_bf16,
                 int32_t batch, int32_t k, int32_t o, int32_t relu, void* stream);

/* Linear layer on the tensor cores (tcgen05, swap-AB: 128 output features x
 * a batch tile of 16..256 rows per UMMA, both operands by TMA), any batch:
 * y[b][o] = act(sum_k x[b][k] * w[o][k] + bias[o]); x bf16 [batch][k],
 * w bf16 [o][k], k % 64 == 0; y fp32 or bf16 (y_bf16). Long-K / few-tile shapes
 * (weight streaming at small batch) split K across CTAs: the partials go to
 * `workspace` (daris_linear_plan().workspace_floats, zero-initialised, left
 * zeroed) with one self-resetting ticket per tile in `counters`. */
typedef struct daris_linear_desc {
  const void* x;
  const void* w;
  const float* bias;      /* [o] or NULL */
  void* y;
  float* workspace;
  int32_t* counters;
  int32_t batch, k, o;
  int32_t relu;           /* 1: ReLU, 0: none */
  int32_t y_bf16;
  int32_t splits;         /* 0 = auto */
  int32_t sm_budget;      /* SMs available to this launch (0 = whole device) */
} daris_linear_desc;

typedef struct daris_linear_plan_t {
  int32_t block_n;        /* batch rows per tile (UMMA N) */
  int32_t splits, kb_per_split, tiles_m, tiles_n;
  int64_t workspace_floats;
  int32_t counters;
  int32_t ctas;
} daris_linear_plan_t;

int daris_linear_plan(const daris_linear_desc* d, daris_linear_plan_t* out);
int daris_linear_tc(const daris_linear_desc* d, void* stream);

/* Global average pooling NHWC bf16 [n][hw][c] -> bf16 [n][c] (feeds daris_linear_tc). */
int daris_avgpool_bf16(const void* x, void* y, int32_t n, int32_t hw, int32_t c, void* stream);

/* Depthwise 3x3 conv + folded BN + ReLU6/ReLU, NHWC bf16, c % 8 == 0,
 * weight [kh][kw][c] bf16. */
int daris_dwconv(const void* x, void* y, const void* weight, const float* scale, const float* bias, int32_t n,
                 int32_t h, int32_t w, int32_t c, int32_t k, int32_t stride, int32_t pad, int32_t ho, int32_t wo,
                 int32_t relu, void* stream);

/* Debug builds (-DDARIS_PAIR_DEBUG) only: host-mapped words where a CTA-pair
 * kernel's mbarrier wait that has not completed after 2 s records its site
 * (word 0: count; words 4..: site | rank << 4 | parity << 5 | blockIdx.x << 8 |
 * blockIdx.y << 20). Returns DARIS_K_BAD_ARG in release builds. */
int daris_debug_pair_watch(void* host_mapped_words);

/* Number of SMs on the current device (cached). */
int daris_device_sms(void);

#ifdef __cplusplus
}
#endif
#endif
