// l3_internal.cuh — device-side building blocks of the B200 L3 decoder.
//
// Product code (sm_100a). Shares nothing with oracle/. The format and the
// arithmetic follow PAPER.md §4.2-§4.3 with the readings of DESIGN.md §3.
#pragma once

#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <stdint.h>

#include "../../include/l3.h"

namespace l3 {

// ---------------------------------------------------------------- tunables
constexpr int kWarpsPerCta = 4;            // decode CTA = 4 warps (128 threads)
constexpr int kSlotBytes = 1024;           // TMA bulk-copy chunk = one ring slot
constexpr int kSlots = 8;                  // ring = 8 KB per warp
constexpr int kRingBytes = kSlotBytes * kSlots;
constexpr int kRingWords = kRingBytes / 4;
constexpr int kMaxRowBytes = (12 + 8 * 255) / 8 + 2;   // one row record never spans more
constexpr uint32_t kNoError = 0xFFFFFFFFu;
constexpr int kMaxUnitsPerImage = 1 << 29;  // 3P must stay below (unit index in error key)

// Per-image descriptor, written by the parse kernel (step a1).
struct ImgDesc {
  uint64_t file_off;   // byte offset of the file in src
  uint64_t data_off;   // byte offset of the data section in src
  uint64_t data_len;   // bytes of the data section
  uint64_t out_off;    // element offset of the [3,H,W] output block
  uint32_t W, H;
  uint32_t N, gx;
  uint32_t P;          // patches per channel
  uint32_t G;          // units (patches) per warp task
  uint32_t L;          // lanes per unit (segment width, power of two)
  uint32_t tasks;      // ceil(3P / G)
  uint32_t mode;       // decode path: 0 whole-staged 4-column lanes (N <= 32), 1 / 2 wide 8-column
                       // lanes with 4 KB / 2 KB segment rings (65..128 / 33..64), 3 generic (N > 128)
  uint32_t cy, cx, ch, cw, flip;   // output window (crop) of the image: rows [cy, cy+ch), cols [cx, cx+cw)
  uint32_t px0, py0, gxw, gyw;     // crop: the patches the window touches, [px0, px0+gxw) x [py0, py0+gyw)
  uint32_t pad_[2];
};
static_assert(sizeof(ImgDesc) == 112, "ImgDesc");

// Workspace layout (256-byte aligned sections).
// Zero-filled before first use; every decode launch leaves it zero-filled again
// (the last CTA resets it), so the workspace is reusable without host work.
struct WsHead {
  unsigned long long next_task[2];   // dynamic schedulers: [0] N <= 128, [1] N > 128
  unsigned int done_ctas;            // last-CTA ticket
  unsigned int pad[59];
};
static_assert(sizeof(WsHead) == 256, "WsHead");

__host__ __device__ inline uint64_t align_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }

struct WsView {
  WsHead* head;
  ImgDesc* desc;          // n
  uint64_t* prefix[2];    // n+1 each: exclusive task prefix per kernel class
  uint32_t* errkey;       // n
  __host__ __device__ static uint64_t bytes(int n) {
    return 256 + align_up(sizeof(ImgDesc) * (uint64_t)n, 256) + 2 * align_up(8ull * (n + 1), 256) +
           align_up(4ull * n, 256);
  }
  __host__ __device__ static WsView at(void* ws, int n) {
    WsView v;
    char* p = (char*)ws;
    v.head = (WsHead*)p; p += 256;
    v.desc = (ImgDesc*)p; p += align_up(sizeof(ImgDesc) * (uint64_t)n, 256);
    v.prefix[0] = (uint64_t*)p; p += align_up(8ull * (n + 1), 256);
    v.prefix[1] = (uint64_t*)p; p += align_up(8ull * (n + 1), 256);
    v.errkey = (uint32_t*)p;
    return v;
  }
};

// Decode path, lanes per unit and units per task for patch size N:
//  * N <= 32: 4 columns per lane, segment = next power of two >= ceil(N/4)
//    lanes, G = 32 / L units per warp, capped so G worst-case patches (+ slack)
//    fit the warp's 8 KB ring (the whole task is staged at once): mode 0;
//  * 33..64: 8 columns per lane, L = 8, G = 4 units, each streamed through its
//    own 2 KB ring: mode 2;
//  * 65..128: 8 columns per lane, L = 16, G = 2 units, 4 KB rings: mode 1;
//  * N > 128 (never chosen by the policy): generic path, one unit per warp,
//    two 128-column chunks per lane: mode 3.
__host__ __device__ inline void lanes_and_group(uint32_t N, uint32_t* L, uint32_t* G, uint32_t* mode) {
  if (N > 128) { *L = 32; *G = 1; *mode = 3; return; }
  if (N > 64) { *L = 16; *G = 2; *mode = 1; return; }
  if (N > 32) { *L = 8; *G = 4; *mode = 2; return; }
  uint32_t need = (N + 3) / 4;
  uint32_t l = 1;
  while (l < need && l < 32) l <<= 1;
  uint32_t g = 32 / l;
  uint64_t worst = ((uint64_t)N * (12 + 8ull * N) + 7) / 8;   // all rows k = 8
  while (g > 1 && g * (worst + 48) > (uint64_t)kRingBytes) g >>= 1;
  *L = l;
  *G = g;
  *mode = 0;
}

// Per-image first-error key, stored complemented so that 0 means "no error": a zero-filled workspace is
// clean with no launch-time initialisation (a1 may run inside the decode CTAs), and the a7 finisher
// re-zeroes each key after reading it. record_err keeps the minimum key (atomicMax of ~key).
__device__ __forceinline__ void record_err(uint32_t* slot, uint32_t key) { atomicMax(slot, ~key); }

// a1 results kept in a decode CTA's shared memory (small batches, no a1 launch): the fields of ImgDesc the
// planar kernels use; data_off is file_off + 13 + 12 P.
struct A1Compact {
  uint64_t file_off, out_off, data_len;
  uint32_t W, H, gx, P;
  uint8_t N, mode, G, L;
  int32_t st;   // header status of a1 (L3_OK or the error)
};
static_assert(sizeof(A1Compact) == 48, "A1Compact");
constexpr int kA1InMaxN = 32;   // batches of up to this many images run a1 inside every decode CTA
__device__ __forceinline__ ImgDesc a1_expand(const A1Compact& c) {
  ImgDesc d = ImgDesc{};
  d.file_off = c.file_off;
  d.data_off = c.file_off + 13ull + 12ull * c.P;
  d.data_len = c.data_len;
  d.out_off = c.out_off;
  d.W = c.W;
  d.H = c.H;
  d.N = c.N;
  d.gx = c.gx;
  d.P = c.P;
  d.G = c.G;
  d.L = c.L;
  d.mode = c.mode;
  return d;
}

// Per-unit half of the a1 offset-table check (the oracle's
// header rule): offsets start at 0, strictly increase over R||G||B and stay inside the data
// section. Unit u checks its own offset and the next one, so a file truncated inside unit u's
// data (off[u+1] >= data_len) is CORRUPT_HEADER for unit u too: its byte range would otherwise
// run past the file (and, for the last file of a batch, past the source buffer).
__device__ __forceinline__ bool unit_offsets_bad(uint32_t u, uint32_t nunits, uint64_t off, uint64_t nxt,
                                                 uint64_t data_len) {
  return (u == 0 && off != 0) || off >= data_len || (u + 1 < nunits && (nxt <= off || nxt >= data_len));
}

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t tx) {
  asm volatile(
      "{\n\t.reg .b64 st;\n\t"
      "mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(smem_u32(bar)),
      "r"(tx)
      : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}

// TMA 1-D bulk copy global -> shared, completion on an mbarrier (sm_90+; UBLKCP in SASS).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ uint32_t bswap32(uint32_t x) { return __byte_perm(x, 0, 0x0123); }

// 32 stream bits starting at bit offset `bit` (MSB-first byte order, reading C8)
// from a ring of little-endian 32-bit words; wraps modulo the ring size.
__device__ __forceinline__ uint32_t ring_bits32(const uint32_t* ring, uint32_t bit) {
  uint32_t wi = bit >> 5;
  uint32_t hi = bswap32(ring[wi & (kRingWords - 1)]);
  uint32_t lo = bswap32(ring[(wi + 1) & (kRingWords - 1)]);
  return __funnelshift_l(lo, hi, bit & 31);
}

// Custom Paeth predictor (Fig. 3): candidate of (TL, T, TR)
// closest to TL + TR - T, ties in the order TL, T, TR (reading C3).
// dTL = |T - TR|, dT = |TL + TR - 2T|, dTR = |TL - T|.
__device__ __forceinline__ int paeth_pred(int tl, int t, int tr) {
  int dtl = __usad(t, tr, 0);
  int dtr = __usad(tl, t, 0);
  int dt = abs(tl + tr - 2 * t);
  int p = (dt <= dtr) ? t : tr;
  return (dtl <= dt && dtl <= dtr) ? tl : p;
}

// ORIGINAL Paeth predictor (PNG): a = left, b = top, c = top-left;
// closest of the three to a + b - c, ties a, b, c. Ablation format variant "L3IP"
// only (reading C16). da = |b - c|, db = |a - c|, dc = |a + b - 2c|.
__device__ __forceinline__ int paeth_png_pred(int a, int b, int c) {
  const int da = __usad(b, c, 0), db = __usad(a, c, 0), dc = abs(a + b - 2 * c);
  if (da <= db && da <= dc) return a;
  return db <= dc ? b : c;
}

// File magic "L3IP" (4th byte 'P') selects the original-Paeth variant.
__device__ __forceinline__ bool is_png_variant(const uint8_t* file) { return file[3] == 'P'; }

}  // namespace l3
