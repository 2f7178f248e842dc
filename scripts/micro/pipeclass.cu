// Which SM pipe does each integer op issue to on sm_100a? One kernel per op (8 independent chains per
// thread); profile with ncu --metrics sm__inst_executed_pipe_alu.sum,sm__inst_executed_pipe_fma.sum,
// sm__inst_executed_pipe_fmaheavy.sum,sm__inst_executed_pipe_fmalite.sum,smsp__inst_executed.sum,...
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define ITER 2048
#define K(name, BODY) \
  __global__ void name(uint32_t* out, uint32_t s) { \
    uint32_t a[8]; for (int i = 0; i < 8; i++) a[i] = threadIdx.x * (i + 3) ^ s; \
    const uint32_t y = s * 7u + 1u, z = s ^ 0x5a5a5a5au; \
    for (int it = 0; it < ITER; it++) { _Pragma("unroll") for (int i = 0; i < 8; i++) { uint32_t x = a[i]; BODY; a[i] = x; } } \
    uint32_t r = 0; for (int i = 0; i < 8; i++) r ^= a[i]; out[blockIdx.x * blockDim.x + threadIdx.x] = r; }
K(k_iadd3, asm volatile("add.u32 %0, %0, %1;" : "+r"(x) : "r"(y)))
K(k_iadd3_3, asm volatile("{.reg .u32 t; add.u32 t, %0, %1; sub.u32 %0, t, %2;}" : "+r"(x) : "r"(y), "r"(z)))
K(k_vmax2, x = __vmaxu2(x, y))
K(k_vmin3, x = __vimin3_u16x2(x, y, z))
K(k_lop3, asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x) : "r"(y), "r"(z)))
K(k_prmt, asm volatile("prmt.b32 %0, %0, %1, 0x3012;" : "+r"(x) : "r"(y)))
K(k_shf, asm volatile("shf.r.clamp.b32 %0, %0, %1, %2;" : "+r"(x) : "r"(y), "r"(z)))
K(k_imad, asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x) : "r"(y), "r"(z)))
K(k_vabs, x = __vabsdiffu4(x, y))
K(k_ffma, asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+r"(x) : "r"(y), "r"(z)))
K(k_sel, asm volatile("{.reg .pred p; setp.lt.u32 p, %1, %2; selp.b32 %0, %0, %1, p;}" : "+r"(x) : "r"(y), "r"(z)))
K(k_imnmx, x = max(x, y))
typedef void (*kf)(uint32_t*, uint32_t);
int main() {
  kf ks[] = {k_iadd3, k_iadd3_3, k_vmax2, k_vmin3, k_lop3, k_prmt, k_shf, k_imad, k_vabs, k_ffma, k_sel, k_imnmx};
  const char* nm[] = {"iadd", "iadd3", "vmax2", "vmin3", "lop3", "prmt", "shf", "imad", "vabsdiff4", "ffma", "setp_sel", "imnmx"};
  uint32_t* out; cudaMalloc(&out, 148 * 8 * 256 * 4);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int i = 0; i < 12; i++) {
    ks[i]<<<148 * 8, 256>>>(out, 1);
    cudaEventRecord(e0); ks[i]<<<148 * 8, 256>>>(out, 1); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double wi = 148.0 * 8 * 8 * ITER * 8;   // warp-level source ops
    printf("%-10s %.2f warp-ops/clk/SM\n", nm[i], wi / (ms * 1e-3 * clk * 1e3) / 148);
  }
  return 0;
}
