// hobf_internal.h -- types shared by the C-ABI layer and the per-format kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace hobf {

// What a conv launcher chose (hobf_conv_kernel_info): filled instead of launching.
struct LaunchInfo {
  const void* func;  // the __global__ function
  int variant;       // schedule (0 for the gate / depthwise kernels)
  int threads;       // threads per CTA
  size_t smem;       // dynamic shared memory bytes
  int64_t blocks;    // CTAs
};

struct ConvArgs {
  const uint32_t* x;   // input planes  [n][h][w][ceil(cin/32)][NPI]
  const uint32_t* wt;  // weight planes [kh][kw][cin][ceil(cout/32)][NPI], or weight tables
  uint32_t* y;         // output planes [n][ho][wo][ceil(cout/32)][NPO]
  int n, h, w, cin, kh, kw, cout, stride, pad, relu, ho, wo;
  int64_t items;       // n * ho * wo * ceil(cout/32)
  int variant;         // kernel variant (0 = auto)
  int out_mode;        // 0: y = output planes F(we, wfo) [pix][G][NPO]
                       // 1: y = planes of the next layer's F(we, next_wf) [pix][G][roundup(3+we+next_wf, 4)]
                       // 2: y = next layer's activation records, F(we, next_wf), [n][cout][ho+2np][wo+2np]
                       // 3: y = float32 NHWC [n][ho][wo][cout], the exact decoded outputs
  int next_wf, next_pad;
  int one;             // always 1 (opaque to the compiler, see bcast_bit)
  unsigned two;        // always 2 (see bit01)
  unsigned row_mul;    // 2^12: IMAD.HI(rec, row_mul) = rec >> 20 (table row of an activation record)
  unsigned lift[32];   // lift[j] = 2^(31-j), runtime values so the multiplies stay IMADs
  int split_e, split_s, split_l;  // variant 12 (fractional wave): extra units, segments per unit, taps per segment
  LaunchInfo* info;    // non-null: record the chosen kernel and launch shape, launch nothing
};

typedef cudaError_t (*conv_launcher)(const ConvArgs&, cudaStream_t);
typedef cudaError_t (*mac_launcher)(uint32_t*, const uint32_t*, const uint32_t*, int64_t, cudaStream_t);

struct FormatEntry {
  int we, wf, rnd, ext, g_mac, g_mul, g_add, g_relu, g_tab;
  conv_launcher conv;
  mac_launcher mac;
  conv_launcher conv_tab;  // conv with the multiplier read from per-weight tables
  conv_launcher conv_dw;   // depthwise conv (full MAC per lane)
};

}  // namespace hobf
