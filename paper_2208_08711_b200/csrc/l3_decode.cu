// l3_decode.cu — sm_100a kernels of the L3 batch decode hot path.
//
//   a1  l3_parse_kernel     header parse + validation + work decomposition
//                           ("first reads the header of each
//                           image and then splits it into multiple patches")
//   a2-a7 l3_decode_kernel  persistent patch decoder: TMA bulk staging of the
//                           compressed unit into a per-warp shared-memory ring
//                           (a2), row-header chain (a3), pixel-parallel delta
//                           unpack (a4), row-parallel custom Paeth
//                           (a5), u8 / fused fp32 store (a6),
//                           first-error status (a7).
//
// Work unit = (image, channel, patch) as in the paper's patch-level parallelism
// (PAPER.md:174), but mapped to a WARP (or a sub-warp segment for N <= 64), not a
// thread block: one lane holds 4 consecutive columns of the patch row, the
// previous row lives in registers and TL/TR neighbours cross lanes by shuffles.
// DESIGN.md §5 explains the mapping and its roofline.
#include <cuda_runtime.h>
#include <stdint.h>

#include "l3_internal.cuh"

namespace l3 {

// ============================================================== a1: parse
struct ParseParams {
  const uint8_t* src;
  const uint64_t* src_offsets;
  const int32_t* shapes;
  const uint64_t* out_offsets;
  int32_t n;
  int32_t* status;
  int32_t* bad_unit;
  WsView ws;
};

__device__ __forceinline__ uint32_t ld_u32le(const uint8_t* p) {
  return (uint32_t)__ldg(p) | ((uint32_t)__ldg(p + 1) << 8) | ((uint32_t)__ldg(p + 2) << 16) |
         ((uint32_t)__ldg(p + 3) << 24);
}

// Block-wide exclusive scan of two u64 values (1024 threads).
__device__ void block_exclusive_scan2(uint64_t& a, uint64_t& b, uint64_t* sh_a, uint64_t* sh_b,
                                      uint64_t& tot_a, uint64_t& tot_b) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint64_t ia = a, ib = b;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    uint64_t ta = __shfl_up_sync(0xffffffffu, ia, d);
    uint64_t tb = __shfl_up_sync(0xffffffffu, ib, d);
    if (lane >= d) { ia += ta; ib += tb; }
  }
  if (lane == 31) { sh_a[wid] = ia; sh_b[wid] = ib; }
  __syncthreads();
  if (wid == 0) {
    uint64_t wa = sh_a[lane], wb = sh_b[lane];
    uint64_t xa = wa, xb = wb;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      uint64_t ta = __shfl_up_sync(0xffffffffu, xa, d);
      uint64_t tb = __shfl_up_sync(0xffffffffu, xb, d);
      if (lane >= d) { xa += ta; xb += tb; }
    }
    sh_a[lane] = xa - wa;   // exclusive warp offsets
    sh_b[lane] = xb - wb;
    if (lane == 31) { sh_a[32] = xa; sh_b[32] = xb; }
  }
  __syncthreads();
  uint64_t ea = ia - a + sh_a[wid], eb = ib - b + sh_b[wid];
  tot_a = sh_a[32];
  tot_b = sh_b[32];
  a = ea;
  b = eb;
  __syncthreads();
}

__global__ void __launch_bounds__(1024) l3_parse_kernel(ParseParams p) {
  __shared__ uint64_t sh_a[33], sh_b[33];
  if (threadIdx.x == 0) {
    p.ws.head->next_task[0] = 0;
    p.ws.head->next_task[1] = 0;
    p.ws.head->done_ctas = 0;
  }
  uint64_t carry0 = 0, carry1 = 0;
  for (int base = 0; base < p.n; base += blockDim.x) {
    const int i = base + threadIdx.x;
    uint64_t t0 = 0, t1 = 0;
    if (i < p.n) {
      const uint64_t f0 = p.src_offsets[i], f1 = p.src_offsets[i + 1];
      const uint64_t len = f1 > f0 ? f1 - f0 : 0;
      const uint8_t* f = p.src + f0;
      int st = L3_OK;
      ImgDesc d = {};
      const int32_t expH = p.shapes[2 * i], expW = p.shapes[2 * i + 1];
      d.out_off = p.out_offsets ? p.out_offsets[i] : (uint64_t)i * 3ull * (uint64_t)expH * (uint64_t)expW;
      if (f1 < f0 || len < 4 || __ldg(f) != 'L' || __ldg(f + 1) != '3' || __ldg(f + 2) != 'I' ||
          __ldg(f + 3) != 'F') {
        st = L3_E_UNRECOGNIZED_FORMAT;
      } else if (len < 13) {
        st = L3_E_CORRUPT_HEADER;
      } else {
        d.W = ld_u32le(f + 4);
        d.H = ld_u32le(f + 8);
        d.N = __ldg(f + 12);
        if (d.W == 0 || d.H == 0 || d.N == 0 || d.W != (uint32_t)expW || d.H != (uint32_t)expH) {
          st = L3_E_CORRUPT_HEADER;
        } else {
          const uint64_t gx = (d.W + d.N - 1) / d.N, gy = (d.H + d.N - 1) / d.N;
          const uint64_t P = gx * gy;
          const uint64_t hdr = 13ull + 12ull * P;
          if (3ull * P >= (uint64_t)kMaxUnitsPerImage || len < hdr) {
            st = L3_E_CORRUPT_HEADER;
          } else {
            d.gx = (uint32_t)gx;
            d.P = (uint32_t)P;
            d.file_off = f0;
            d.data_off = f0 + hdr;
            d.data_len = len - hdr;
            lanes_and_group(d.N, &d.L, &d.G);
            d.tasks = (uint32_t)((3ull * P + d.G - 1) / d.G);
            if (d.N <= 128) t0 = d.tasks; else t1 = d.tasks;
          }
        }
      }
      if (st != L3_OK) d.tasks = 0;
      p.ws.desc[i] = d;
      p.ws.errkey[i] = kNoError;
      p.status[i] = st;
      if (p.bad_unit) p.bad_unit[i] = -1;
    }
    uint64_t tot0, tot1;
    block_exclusive_scan2(t0, t1, sh_a, sh_b, tot0, tot1);
    if (i < p.n) {
      p.ws.prefix[0][i] = carry0 + t0;
      p.ws.prefix[1][i] = carry1 + t1;
    }
    carry0 += tot0;
    carry1 += tot1;
  }
  if (threadIdx.x == 0) {
    p.ws.prefix[0][p.n] = carry0;
    p.ws.prefix[1][p.n] = carry1;
  }
}

// ============================================================== a2-a7: decode
struct DecodeParams {
  const uint8_t* src;
  uint64_t src_total;       // src_offsets[n] read on device (see kernel)
  const uint64_t* src_offsets;
  int32_t n;
  void* out;
  float scale[3], bias[3];
  int32_t* status;
  int32_t* bad_unit;
  WsView ws;
  int cls;                  // 0: N <= 128 tasks, 1: N > 128 tasks
  int finalize;             // last CTA writes status / bad_unit
  uint32_t key_scale;       // 128: predictor key scale, passed at run time (keeps key math on IMAD)
};

__device__ __forceinline__ uint32_t err_key(uint32_t unit, int code) {
  return 0x80000000u | (unit << 1) | (code == L3_E_TRUNCATED_STREAM ? 1u : 0u);
}

// Upper bound of the bytes a w x h patch can occupy (every row k = 8).
__device__ __forceinline__ uint32_t worst_patch_bytes(uint32_t w, uint32_t h) {
  return (h * (12u + 8u * w) + 7u) / 8u;
}

// Stage src[a, b) (absolute byte offsets) into ring bytes starting at dst16
// (16-byte aligned); `a16` = a rounded down to 16. The part below `lim` (the
// batch end rounded down to 16) moves with one TMA bulk copy completing on
// `bar`; the remaining < 16 tail bytes are copied by the segment's lanes.
// Returns the number of bulk bytes (already armed on the barrier by lane `leader`).
__device__ __forceinline__ void stage_range(const uint8_t* src, uint64_t a16, uint64_t b16, uint64_t lim,
                                            uint64_t real_end, uint8_t* dst16, uint64_t* bar, bool leader,
                                            int seg_lane, int seg_lanes) {
  uint64_t bulk_end = b16 < lim ? b16 : lim;
  uint32_t bulk = bulk_end > a16 ? (uint32_t)(bulk_end - a16) : 0u;
  if (leader) {
    mbar_arrive_expect_tx(bar, bulk);
    if (bulk) bulk_g2s(dst16, src + a16, bulk, bar);
  }
  // tail: bytes in [max(a16, lim), real_end) that the bulk copy could not move
  uint64_t t0 = a16 > lim ? a16 : lim;
  for (uint64_t x = t0 + seg_lane; x < real_end && x < b16; x += seg_lanes) dst16[x - a16] = __ldg(src + x);
}

template <int MAXCH, bool F32>
__global__ void __launch_bounds__(kWarpsPerCta * 32)
    l3_decode_kernel(DecodeParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* ring8 = smem + warp * kRingBytes;
  const uint32_t* ring = reinterpret_cast<const uint32_t*>(ring8);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kWarpsPerCta * kRingBytes) + warp * kSlots;
  if (lane == 0) {
    for (int s = 0; s < kSlots; s++) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncwarp();
  uint32_t phase_bits = 0;   // per-slot parity of the next phase to wait for

  const uint64_t* prefix = p.cls ? p.ws.prefix[1] : p.ws.prefix[0];
  const uint64_t total_tasks = prefix[p.n];
  const uint64_t src_total = p.src_offsets[p.n];
  const uint64_t lim = src_total & ~15ull;

  for (;;) {
    uint64_t task = 0;
    if (lane == 0) task = atomicAdd(p.cls ? &p.ws.head->next_task[1] : &p.ws.head->next_task[0], 1ull);
    task = __shfl_sync(0xffffffffu, task, 0);
    if (task >= total_tasks) break;
    // image of this task: last i with prefix[i] <= task (images with 0 tasks are skipped)
    int lo = 0, hi = p.n;   // prefix[lo] <= task < prefix[hi]
    while (hi - lo > 1) {
      int mid = (lo + hi) >> 1;
      if (__ldg(&prefix[mid]) <= task) lo = mid; else hi = mid;
    }
    const int img = lo;
    const ImgDesc d = p.ws.desc[img];
    const uint32_t t = (uint32_t)(task - prefix[img]);
    const uint32_t L = d.L, G = d.G;
    const uint32_t seg = lane / L, j = lane % L;
    const uint32_t nunits = 3u * d.P;
    const uint32_t u = t * G + seg;
    const uint8_t* file = p.src + d.file_off;

    // ---- unit geometry and byte range (a1 remainder: this unit's offsets)
    bool active = (seg < G) && (u < nunits);
    uint32_t w = 0, h = 0, x0 = 0, y0 = 0, ch = 0;
    uint64_t start = 0, end = 0;
    if (active) {
      ch = u / d.P;
      const uint32_t pp = u - ch * d.P;
      const uint32_t px = pp % d.gx, py = pp / d.gx;
      x0 = px * d.N;
      y0 = py * d.N;
      w = min(d.N, d.W - x0);
      h = min(d.N, d.H - y0);
      const uint64_t off = ld_u32le(file + 13 + 4ull * u);
      const uint64_t nxt = (u + 1 < nunits) ? (uint64_t)ld_u32le(file + 17 + 4ull * u) : d.data_len;
      if ((u == 0 && off != 0) || off >= d.data_len || (u + 1 < nunits && nxt <= off)) {
        if (j == 0) atomicMin(&p.ws.errkey[img], 0u);   // header-level: CORRUPT_HEADER
        active = false;
      } else {
        start = d.data_off + off;
        end = d.data_off + nxt;
      }
    }
    // staging window: never more than the worst-case patch (+ slack for the
    // 32-bit read window); bytes past it are never read by a valid stream.
    const uint32_t worst = active ? worst_patch_bytes(w, h) : 0u;
    const uint64_t stage_end = active ? min(end, start + worst + 8) : 0;
    const uint32_t len_bits = active ? (uint32_t)min((uint64_t)(worst + 16), end - start) * 8u : 0u;

    uint32_t bitpos = 0;   // ring-relative bit position of the unit's next row record
    const bool stream = (G == 1);
    uint32_t nchunks = 0, issued = 0, landed = 0;
    uint64_t A = 0;
    if (!stream) {
      // ---- whole-task staging: one aligned window per segment, one barrier
      const uint32_t seg_bytes = kRingBytes / G;   // >= worst + 32 by construction (lanes_and_group)
      uint32_t bytes = 0;
      uint64_t a16 = 0, b16 = 0;
      if (active) {
        a16 = start & ~15ull;
        b16 = (stage_end + 15) & ~15ull;
        const uint64_t be = b16 < lim ? b16 : lim;
        bytes = be > a16 ? (uint32_t)(be - a16) : 0u;
        bitpos = seg * seg_bytes * 8u + (uint32_t)(start - a16) * 8u;
      }
      // total tx for barrier 0 = sum over segments (count only segment leaders)
      uint32_t tx = (active && j == 0) ? bytes : 0u;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) tx += __shfl_xor_sync(0xffffffffu, tx, o);
      if (lane == 0) mbar_arrive_expect_tx(&bars[0], tx);
      __syncwarp();
      if (active) {
        uint8_t* dst = ring8 + seg * seg_bytes;
        if (j == 0 && bytes) bulk_g2s(dst, p.src + a16, bytes, &bars[0]);
        const uint64_t t0 = a16 > lim ? a16 : lim;
        for (uint64_t x = t0 + j; x < stage_end && x < b16; x += L) dst[x - a16] = __ldg(p.src + x);
      }
      mbar_wait(&bars[0], phase_bits & 1u);
      phase_bits ^= 1u;
      __syncwarp();
    } else {
      // ---- streaming through the ring: chunk i of [A, B) -> slot i % kSlots
      if (active) {
        A = start & ~15ull;
        const uint64_t B = (stage_end + 15) & ~15ull;
        nchunks = (uint32_t)((B - A + kSlotBytes - 1) / kSlotBytes);
        bitpos = (uint32_t)(start - A) * 8u;
        const uint32_t first = min(nchunks, (uint32_t)kSlots);
        for (uint32_t c = 0; c < first; c++) {
          const uint64_t ca = A + (uint64_t)c * kSlotBytes;
          const uint64_t cb = min(ca + kSlotBytes, B);
          stage_range(p.src, ca, cb, lim, stage_end, ring8 + (c % kSlots) * kSlotBytes, &bars[c % kSlots],
                      lane == 0, lane, 32);
        }
        issued = first;
      }
      __syncwarp();
    }
    const uint32_t seg_bit0 = bitpos;

    // ---- row loop (a3-a6): rows are sequential, columns parallel
    uint32_t hmax = active ? h : 0u;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) hmax = max(hmax, __shfl_xor_sync(0xffffffffu, hmax, o));

    const uint64_t plane = d.out_off + (uint64_t)ch * d.W * d.H;
    const float sc = F32 ? (ch == 0 ? p.scale[0] : (ch == 1 ? p.scale[1] : p.scale[2])) : 0.f;
    const float bi = F32 ? (ch == 0 ? p.bias[0] : (ch == 1 ? p.bias[1] : p.bias[2])) : 0.f;
    int prev[MAXCH][4];
#pragma unroll
    for (int q = 0; q < MAXCH; q++)
#pragma unroll
      for (int s = 0; s < 4; s++) prev[q][s] = 0;
    bool dead = !active;
    const uint32_t row_bytes_max = (12u + 8u * w) / 8u + 8u;

    for (uint32_t r = 0; r < hmax; r++) {
      if (stream && active) {
        // make sure every chunk this row can touch has landed (warp-uniform: G == 1)
        const uint32_t need_byte = (bitpos >> 3) + row_bytes_max;
        const uint32_t c_need = min(need_byte / kSlotBytes, nchunks - 1);
        while (landed <= c_need) {
          const uint32_t s = landed % kSlots;
          mbar_wait(&bars[s], (phase_bits >> s) & 1u);
          phase_bits ^= 1u << s;
          landed++;
        }
      }
      bool live = !dead && r < h;
      uint32_t k = 0, base = 0;
      if (live) {
        const uint32_t avail = len_bits - (bitpos - seg_bit0);
        const uint32_t hdr = ring_bits32(ring, bitpos);
        k = hdr >> 28;
        base = (hdr >> 20) & 0xFFu;
        int code = L3_OK;
        if (avail < 4) code = L3_E_TRUNCATED_STREAM;
        else if (k == 0 || k > 8) code = L3_E_CORRUPT_STREAM;
        else if (avail < 12u + k * w) code = L3_E_TRUNCATED_STREAM;
        if (code != L3_OK) {
          if (j == 0) atomicMin(&p.ws.errkey[img], err_key(u, code));
          dead = true;
          live = false;
        }
      }
      // a4: pixel-wise delta unpack -> res = base + delta
      int res[MAXCH][4];
#pragma unroll
      for (int q = 0; q < MAXCH; q++) {
        const uint32_t c = q * 128u + 4u * j;
        uint32_t field = 0;
        if (live && c < w) field = ring_bits32(ring, bitpos + 12u + c * k);
#pragma unroll
        for (int s = 0; s < 4; s++) res[q][s] = (int)(base + ((field << (k * s)) >> (32 - k)));
      }
      // a5: row-parallel custom Paeth against the previous row
      int pix[MAXCH][4];
      if (r == 0) {
#pragma unroll
        for (int q = 0; q < MAXCH; q++)
#pragma unroll
          for (int s = 0; s < 4; s++) pix[q][s] = res[q][s] & 0xFF;
      } else {
        int left[MAXCH], right[MAXCH];
#pragma unroll
        for (int q = 0; q < MAXCH; q++) {
          left[q] = __shfl_up_sync(0xffffffffu, prev[q][3], 1, L);
          right[q] = __shfl_down_sync(0xffffffffu, prev[q][0], 1, L);
        }
        if (MAXCH == 2) {
          const int l1 = __shfl_sync(0xffffffffu, prev[0][3], 31);
          const int r0 = __shfl_sync(0xffffffffu, prev[MAXCH - 1][0], 0);
          if (j == 0) left[MAXCH - 1] = l1;
          if (j == 31) right[0] = r0;
        }
#pragma unroll
        for (int q = 0; q < MAXCH; q++) {
          const uint32_t c = q * 128u + 4u * j;
#pragma unroll
          for (int s = 0; s < 4; s++) {
            const int tt = prev[q][s];
            const int tl = (s > 0) ? prev[q][s - 1] : (c > 0 ? left[q] : tt);
            int tr = (s < 3) ? prev[q][s + 1] : right[q];
            if (c + s + 1 >= w) tr = tt;
            pix[q][s] = (paeth_pred(tl, tt, tr) + res[q][s]) & 0xFF;
          }
        }
      }
      // a6: store (u8 planar, or fused cast + normalise to fp32)
      if (live) {
        const uint64_t row_off = plane + (uint64_t)(y0 + r) * d.W + x0;
#pragma unroll
        for (int q = 0; q < MAXCH; q++) {
          const uint32_t c = q * 128u + 4u * j;
          if (c >= w) continue;
          const uint64_t e = row_off + c;
          if (F32) {
            float* o = reinterpret_cast<float*>(p.out) + e;
            float v0 = fmaf((float)pix[q][0], sc, bi), v1 = fmaf((float)pix[q][1], sc, bi);
            float v2 = fmaf((float)pix[q][2], sc, bi), v3 = fmaf((float)pix[q][3], sc, bi);
            if (c + 4 <= w && ((reinterpret_cast<uintptr_t>(o) & 15) == 0)) {
              *reinterpret_cast<float4*>(o) = make_float4(v0, v1, v2, v3);
            } else {
              o[0] = v0;
              if (c + 1 < w) o[1] = v1;
              if (c + 2 < w) o[2] = v2;
              if (c + 3 < w) o[3] = v3;
            }
          } else {
            uint8_t* o = reinterpret_cast<uint8_t*>(p.out) + e;
            if (c + 4 <= w && ((reinterpret_cast<uintptr_t>(o) & 3) == 0)) {
              *reinterpret_cast<uint32_t*>(o) =
                  (uint32_t)pix[q][0] | ((uint32_t)pix[q][1] << 8) | ((uint32_t)pix[q][2] << 16) |
                  ((uint32_t)pix[q][3] << 24);
            } else {
              o[0] = (uint8_t)pix[q][0];
              if (c + 1 < w) o[1] = (uint8_t)pix[q][1];
              if (c + 2 < w) o[2] = (uint8_t)pix[q][2];
              if (c + 3 < w) o[3] = (uint8_t)pix[q][3];
            }
          }
        }
#pragma unroll
        for (int q = 0; q < MAXCH; q++)
#pragma unroll
          for (int s = 0; s < 4; s++) prev[q][s] = pix[q][s];
        bitpos += 12u + k * w;
      }
      if (stream && active) {
        // refill slots whose chunk lies entirely before the current position
        const uint32_t consumed = (bitpos >> 3) / kSlotBytes;
        if (issued < nchunks && issued < consumed + kSlots) {
          __syncwarp();
          fence_proxy_async_smem();
          while (issued < nchunks && issued < consumed + kSlots) {
            const uint64_t ca = A + (uint64_t)issued * kSlotBytes;
            const uint64_t B = (stage_end + 15) & ~15ull;
            const uint64_t cb = min(ca + kSlotBytes, B);
            stage_range(p.src, ca, cb, lim, stage_end, ring8 + (issued % kSlots) * kSlotBytes,
                        &bars[issued % kSlots], lane == 0, lane, 32);
            issued++;
          }
          __syncwarp();
        }
      }
    }
    // drain chunks that were issued but never waited for (early error exit)
    if (stream) {
      while (landed < issued) {
        const uint32_t s = landed % kSlots;
        mbar_wait(&bars[s], (phase_bits >> s) & 1u);
        phase_bits ^= 1u << s;
        landed++;
      }
    }
    __syncwarp();
    fence_proxy_async_smem();
  }

  // ---- a7: per-image status, written by the last CTA of the finishing kernel
  if (p.finalize) {
    __shared__ unsigned int ticket;
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      ticket = atomicAdd(&p.ws.head->done_ctas, 1u);
    }
    __syncthreads();
    if (ticket == gridDim.x - 1) {
      __threadfence();
      for (int i = threadIdx.x; i < p.n; i += blockDim.x) {
        if (p.status[i] != L3_OK) continue;   // header-level error from a1
        const uint32_t key = atomicAdd(&p.ws.errkey[i], 0u);
        if (key == kNoError) continue;
        if (key == 0u) {
          p.status[i] = L3_E_CORRUPT_HEADER;
        } else {
          p.status[i] = (key & 1u) ? L3_E_TRUNCATED_STREAM : L3_E_CORRUPT_STREAM;
          if (p.bad_unit) p.bad_unit[i] = (int32_t)((key >> 1) & 0x3FFFFFFFu);
        }
      }
    }
  }
}

}  // namespace l3

#include "l3_decode_fast.cuh"

namespace l3 {

// Exhaustive self-test of the pair-form predictor used by the fast kernel:
// out[TL<<16 | T<<8 | TR] = paeth_pred2 result, two triples per thread.
__global__ void l3_selftest_paeth_kernel(uint8_t* out, uint32_t K) {
  const uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) * 2u;
  if (i >= (1u << 24)) return;
  const uint32_t a = i, b = i + 1;
  const uint32_t tl = ((a >> 16) & 0xFFu) | (((b >> 16) & 0xFFu) << 16);
  const uint32_t t = ((a >> 8) & 0xFFu) | (((b >> 8) & 0xFFu) << 16);
  const uint32_t tr = (a & 0xFFu) | ((b & 0xFFu) << 16);
  const uint32_t p2 = paeth_pred2(tl, t, tr, K);
  out[a] = (uint8_t)(p2 & 0xFFu);
  out[b] = (uint8_t)((p2 >> 16) & 0xFFu);
  if ((p2 & 0xFF00FF00u) != 0u) out[a] = out[b] = 0xEE;   // pair form must keep bytes 1, 3 zero
}

cudaError_t launch_selftest_paeth(uint8_t* out, cudaStream_t s) {
  l3_selftest_paeth_kernel<<<(1u << 23) / 256, 256, 0, s>>>(out, 128u);
  return cudaGetLastError();
}

// ============================================================== host launch
static int g_sm_count = 0;
static int g_occ[2][2] = {{0, 0}, {0, 0}};

static size_t decode_smem_bytes() { return (size_t)kWarpsPerCta * (kRingBytes + kSlots * 8); }

template <int MAXCH, bool F32>
static cudaError_t launch_decode(const DecodeParams& dp, int grid, cudaStream_t s) {
  auto kern = l3_decode_kernel<MAXCH, F32>;
  const size_t smem = decode_smem_bytes();
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  kern<<<grid, kWarpsPerCta * 32, smem, s>>>(dp);
  return cudaGetLastError();
}

template <int MAXCH, bool F32>
static int occupancy() {
  int occ = 0;
  cudaFuncSetAttribute(l3_decode_kernel<MAXCH, F32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)decode_smem_bytes());
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, l3_decode_kernel<MAXCH, F32>, kWarpsPerCta * 32,
                                                decode_smem_bytes());
  return occ > 0 ? occ : 1;
}

template <bool F32>
static int fast_occupancy() {
  int occ = 0;
  cudaFuncSetAttribute(l3_decode_fast_kernel<F32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)fast_smem_bytes());
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, l3_decode_fast_kernel<F32>, kWarpsPerCta * 32,
                                                fast_smem_bytes());
  return occ > 0 ? occ : 1;
}

template <bool F32>
static cudaError_t launch_fast(const DecodeParams& dp, int grid, cudaStream_t s) {
  l3_decode_fast_kernel<F32><<<grid, kWarpsPerCta * 32, fast_smem_bytes(), s>>>(dp);
  return cudaGetLastError();
}

cudaError_t ensure_device_info() {
  if (g_sm_count == 0) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    e = cudaDeviceGetAttribute(&g_sm_count, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) return e;
    g_occ[0][0] = fast_occupancy<false>();
    g_occ[0][1] = fast_occupancy<true>();
    g_occ[1][0] = occupancy<2, false>();
    g_occ[1][1] = occupancy<2, true>();
  }
  return cudaSuccess;
}

cudaError_t launch_parse(const l3_decode_args* a, cudaStream_t s) {
  ParseParams pp;
  pp.src = a->src;
  pp.src_offsets = a->src_offsets;
  pp.shapes = a->shapes;
  pp.out_offsets = a->out_offsets;
  pp.n = a->n;
  pp.status = a->status;
  pp.bad_unit = a->bad_unit;
  pp.ws = WsView::at(a->workspace, a->n);
  l3_parse_kernel<<<1, 1024, 0, s>>>(pp);
  return cudaGetLastError();
}

cudaError_t launch_decode_units(const l3_decode_args* a, cudaStream_t s) {
  cudaError_t e = ensure_device_info();
  if (e != cudaSuccess) return e;
  DecodeParams dp;
  dp.src = a->src;
  dp.src_total = 0;
  dp.src_offsets = a->src_offsets;
  dp.n = a->n;
  dp.out = a->out;
  for (int c = 0; c < 3; c++) {
    dp.scale[c] = a->scale[c];
    dp.bias[c] = a->bias[c];
  }
  dp.status = a->status;
  dp.bad_unit = a->bad_unit;
  dp.ws = WsView::at(a->workspace, a->n);
  dp.key_scale = 128u;
  const bool f32 = a->out_kind == L3_OUT_F32;
  // class 0: N <= 128, persistent grid = SMs x resident CTAs
  dp.cls = 0;
  dp.finalize = 0;
  const int grid0 = g_sm_count * g_occ[0][f32 ? 1 : 0];
  e = f32 ? launch_fast<true>(dp, grid0, s) : launch_fast<false>(dp, grid0, s);
  if (e != cudaSuccess) return e;
  // class 1: N > 128 (rare; exits at once when there are none) + a7 finalisation
  dp.cls = 1;
  dp.finalize = 1;
  const int grid1 = g_sm_count;
  e = f32 ? launch_decode<2, true>(dp, grid1, s) : launch_decode<2, false>(dp, grid1, s);
  return e;
}

}  // namespace l3
