// Issue-throughput microbenchmark of the integer ops the decode row step uses (sm_100a):
// which ones share the half-rate ALU pipe and which run on the FMA pipe. Each kernel runs
// ITER iterations of 8 independent dependency chains per thread; 148 x 8 CTAs x 256 threads.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define ITER 4096
#define OP_SHF(x, y)  asm volatile("shf.r.clamp.b32 %0, %0, %1, %2;" : "+r"(x) : "r"(y), "r"(y))
#define OP_LOP(x, y)  asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x) : "r"(y), "r"(y ^ 7u))
#define OP_PRMT(x, y) asm volatile("prmt.b32 %0, %0, %1, 0x3012;" : "+r"(x) : "r"(y))
#define OP_IMAD(x, y) asm volatile("mad.lo.u32 %0, %0, %1, %1;" : "+r"(x) : "r"(y))
#define OP_IMADHI(x, y) asm volatile("mul.hi.u32 %0, %0, %1;" : "+r"(x) : "r"(y))
#define OP_VABS(x, y) x = __vabsdiffu4(x, y)
#define OP_VMIN3(x, y) x = __vimin3_u16x2(x, y, y ^ 0x55u)
#define OP_VMAX2(x, y) x = __vmaxu2(x, y)
#define OP_IADD3(x, y) asm volatile("{.reg .u32 t; add.u32 t, %0, %1; add.u32 %0, t, %2;}" : "+r"(x) : "r"(y), "r"(y + 3u))
#define OP_IADD(x, y) asm volatile("add.u32 %0, %0, %1;" : "+r"(x) : "r"(y))
#define OP_ADDIMM(x, y) asm volatile("add.u32 %0, %0, 0x12345;" : "+r"(x))
#define OP_SHL_IMM(x, y) asm volatile("shl.b32 %0, %0, 3;" : "+r"(x))
#define OP_FFMA(x, y) asm volatile("fma.rn.f32 %0, %0, %1, %1;" : "+r"(x) : "r"(y))
#define OP_I2F(x, y) asm volatile("{.reg .f32 f; cvt.rn.f32.u8 f, %0; mov.b32 %0, f;}" : "+r"(x))
#define OP_SEL(x, y) asm volatile("{.reg .pred p; setp.lt.u32 p, %1, 5; selp.b32 %0, %0, %1, p;}" : "+r"(x) : "r"(y))

#define KERNEL(name, OPA, OPB)                                                   \
  __global__ void name(uint32_t* out, uint32_t seed) {                           \
    uint32_t a0 = threadIdx.x ^ seed, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;     \
    uint32_t a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;                 \
    const uint32_t y = seed * 3u + 1u;                                           \
    for (int i = 0; i < ITER; i++) {                                             \
      OPA(a0, y); OPB(a1, y); OPA(a2, y); OPB(a3, y);                            \
      OPA(a4, y); OPB(a5, y); OPA(a6, y); OPB(a7, y);                            \
    }                                                                            \
    out[blockIdx.x * blockDim.x + threadIdx.x] = a0 ^ a1 ^ a2 ^ a3 ^ a4 ^ a5 ^ a6 ^ a7; \
  }

KERNEL(k_shf, OP_SHF, OP_SHF)
KERNEL(k_lop, OP_LOP, OP_LOP)
KERNEL(k_prmt, OP_PRMT, OP_PRMT)
KERNEL(k_imad, OP_IMAD, OP_IMAD)
KERNEL(k_imadhi, OP_IMADHI, OP_IMADHI)
KERNEL(k_vabs, OP_VABS, OP_VABS)
KERNEL(k_vmin3, OP_VMIN3, OP_VMIN3)
KERNEL(k_vmax2, OP_VMAX2, OP_VMAX2)
KERNEL(k_iadd, OP_IADD, OP_IADD)
KERNEL(k_shlimm, OP_SHL_IMM, OP_SHL_IMM)
KERNEL(k_ffma, OP_FFMA, OP_FFMA)
KERNEL(k_i2f, OP_I2F, OP_I2F)
KERNEL(k_sel, OP_SEL, OP_SEL)
KERNEL(k_shf_imad, OP_SHF, OP_IMAD)
KERNEL(k_prmt_imad, OP_PRMT, OP_IMAD)
KERNEL(k_lop_imad, OP_LOP, OP_IMAD)
KERNEL(k_vabs_imad, OP_VABS, OP_IMAD)
KERNEL(k_prmt_lop, OP_PRMT, OP_LOP)
KERNEL(k_prmt_vabs, OP_PRMT, OP_VABS)
KERNEL(k_iadd_lop, OP_IADD, OP_LOP)
KERNEL(k_iadd_imad, OP_IADD, OP_IMAD)
KERNEL(k_ffma_imad, OP_FFMA, OP_IMAD)
KERNEL(k_ffma_lop, OP_FFMA, OP_LOP)
KERNEL(k_imadhi_lop, OP_IMADHI, OP_LOP)
KERNEL(k_shlimm_lop, OP_SHL_IMM, OP_LOP)
KERNEL(k_shlimm_imad, OP_SHL_IMM, OP_IMAD)
KERNEL(k_i2f_lop, OP_I2F, OP_LOP)
KERNEL(k_sel_imad, OP_SEL, OP_IMAD)





typedef void (*kfn)(uint32_t*, uint32_t);
int main() {
  struct { const char* n; kfn f; } ks[] = {
      {"SHF", k_shf}, {"LOP3", k_lop}, {"PRMT", k_prmt}, {"IMAD", k_imad}, {"IMAD.HI", k_imadhi},
      {"VABSDIFF4", k_vabs}, {"VIMNMX3.U16x2", k_vmin3}, {"VIMNMX.U16x2", k_vmax2}, {"IADD(add.u32)", k_iadd},
      {"SHL imm", k_shlimm}, {"FFMA", k_ffma}, {"I2F.U8", k_i2f}, {"SETP+SEL", k_sel},
      {"SHF+IMAD", k_shf_imad}, {"PRMT+IMAD", k_prmt_imad}, {"LOP3+IMAD", k_lop_imad}, {"VABS+IMAD", k_vabs_imad},
      {"PRMT+LOP3", k_prmt_lop}, {"PRMT+VABS", k_prmt_vabs}, {"IADD+LOP3", k_iadd_lop}, {"IADD+IMAD", k_iadd_imad},
      {"FFMA+IMAD", k_ffma_imad}, {"FFMA+LOP3", k_ffma_lop}, {"IMAD.HI+LOP3", k_imadhi_lop},
      {"SHLimm+LOP3", k_shlimm_lop}, {"SHLimm+IMAD", k_shlimm_imad}, {"I2F+LOP3", k_i2f_lop}, {"SETP/SEL+IMAD", k_sel_imad}};
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int blocks = sms * 8, threads = 256;
  uint32_t* out;
  cudaMalloc(&out, blocks * threads * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  printf("SMs %d, clock %d MHz; warp-instructions per clock per SM (4 SMSPs; 4.0 = one per SMSP per clock)\n", sms, clk / 1000);
  for (auto& k : ks) {
    k.f<<<blocks, threads>>>(out, 1);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; r++) k.f<<<blocks, threads>>>(out, 1);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double warp_instr = 5.0 * blocks * (threads / 32) * (double)ITER * 8;   // source ops (may be >1 SASS)
    const double clocks = ms * 1e-3 * clk * 1e3;
    printf("%-16s %6.2f\n", k.n, warp_instr / clocks / sms);
  }
  return 0;
}
