// hobf_lop3.cuh -- the single "cell" of the B200 cell library: PTX lop3.b32.
//
// The paper maps its FP cores onto one Liberty cell per target bitwise
// instruction; for AVX512 that is all 256 three-input functions
// (vpternlog, Table 2 LUT000..LUT255).  lop3.b32 is the same function family
// with the same immediate convention (a = 0xF0, b = 0xCC, c = 0xAA), executed
// on one 32-bit register = one bit of 32 lanes.
#pragma once
#include <stdint.h>

template <unsigned IMM>
__device__ __forceinline__ uint32_t hobf_lop3(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, %4;" : "=r"(d) : "r"(a), "r"(b), "r"(c), "n"(IMM));
  return d;
}
