// Pipe and rate of the packed-half ops (HADD2 / HFMA2 / HMUL2, .SAT, |x| modifiers, HADD2.F32
// conversion) and the int->float converts on sm_100a, for an fp16x2 formulation of the custom Paeth
// predictor. Same harness as pipeclass.cu: one kernel per op, 8 independent chains per thread; the
// event-timed rate, then ncu pipe counters on the same kernels (pipehalf.sh).
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#define ITER 2048
#define K(name, BODY) \
  __global__ void name(uint32_t* out, uint32_t s) { \
    uint32_t a[8]; for (int i = 0; i < 8; i++) a[i] = (threadIdx.x * (i + 3) ^ s) & 0x00FF00FFu | 0x64006400u; \
    const uint32_t y = (s * 7u + 1u) & 0x00FF00FFu | 0x64006400u, z = (s ^ 0x5a5a5a5au) & 0x00FF00FFu | 0x64006400u; \
    for (int it = 0; it < ITER; it++) { _Pragma("unroll") for (int i = 0; i < 8; i++) { uint32_t x = a[i]; BODY; a[i] = x; } } \
    uint32_t r = 0; for (int i = 0; i < 8; i++) r ^= a[i]; out[blockIdx.x * blockDim.x + threadIdx.x] = r; }
K(k_hadd2, asm volatile("add.f16x2 %0, %0, %1;" : "+r"(x) : "r"(y)))
K(k_hfma2, asm volatile("fma.rn.f16x2 %0, %0, %1, %2;" : "+r"(x) : "r"(y), "r"(z)))
K(k_hmul2, asm volatile("mul.f16x2 %0, %0, %1;" : "+r"(x) : "r"(y)))
K(k_hsat_abs, asm volatile("{.reg .b32 t, u; abs.f16x2 t, %0; abs.f16x2 u, %1; sub.sat.f16x2 %0, t, u;}" : "+r"(x) : "r"(y)))
K(k_cvt_f32, asm volatile("{.reg .f32 f; .reg .b16 h, l; mov.b32 {l, h}, %0; cvt.f32.f16 f, l; mov.b32 %0, f;}" : "+r"(x)))
K(k_i2fp, asm volatile("cvt.rn.f32.u32 %0, %0;" : "+r"(x)))
K(k_i2f_u8, asm volatile("{.reg .f32 f; .reg .u8 b; cvt.u8.u32 b, %0; cvt.rn.f32.u8 f, b; mov.b32 %0, f;}" : "+r"(x)))
K(k_ffma, asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+r"(x) : "r"(y), "r"(z)))
K(k_mix_ffma_hfma2, if (i & 1) asm volatile("fma.rn.f16x2 %0, %0, %1, %2;" : "+r"(x) : "r"(y), "r"(z)); else asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+r"(x) : "r"(y), "r"(z)))
K(k_mix_imad_hfma2, if (i & 1) asm volatile("fma.rn.f16x2 %0, %0, %1, %2;" : "+r"(x) : "r"(y), "r"(z)); else asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x) : "r"(y), "r"(z)))
K(k_mix_lop3_hfma2, if (i & 1) asm volatile("fma.rn.f16x2 %0, %0, %1, %2;" : "+r"(x) : "r"(y), "r"(z)); else asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x) : "r"(y), "r"(z)))
K(k_mix_lop3_imad, if (i & 1) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x) : "r"(y), "r"(z)); else asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x) : "r"(y), "r"(z)))
K(k_hmnmx2, asm volatile("min.f16x2 %0, %0, %1;" : "+r"(x) : "r"(y)))
typedef void (*kf)(uint32_t*, uint32_t);
int main() {
  kf ks[] = {k_hadd2, k_hfma2, k_hmul2, k_hsat_abs, k_cvt_f32, k_i2fp, k_i2f_u8, k_ffma, k_mix_ffma_hfma2,
             k_mix_imad_hfma2, k_mix_lop3_hfma2, k_mix_lop3_imad, k_hmnmx2};
  const char* nm[] = {"hadd2", "hfma2", "hmul2", "hsub_sat_abs", "cvt_f32_f16", "i2fp_u32", "i2f_u8", "ffma",
                      "mix_ffma_hfma2", "mix_imad_hfma2", "mix_lop3_hfma2", "mix_lop3_imad", "hmnmx2"};
  const int nk = sizeof(ks) / sizeof(ks[0]);
  uint32_t* out; cudaMalloc(&out, 148 * 8 * 256 * 4);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int i = 0; i < nk; i++) {
    ks[i]<<<148 * 8, 256>>>(out, 1);
    cudaEventRecord(e0); ks[i]<<<148 * 8, 256>>>(out, 1); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double wi = 148.0 * 8 * 8 * ITER * 8;   // warp-level source ops
    printf("%-16s %.2f warp-ops/clk/SM\n", nm[i], wi / (ms * 1e-3 * clk * 1e3) / 148);
  }
  return 0;
}
