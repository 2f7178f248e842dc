// l3_decode_fast.cuh — the hot decode kernel for patch sizes N <= 128 (every
// policy-chosen N). Included by l3_decode.cu.
//
// Same unit mapping as the generic kernel (one warp, or an L-lane segment of it,
// per (image, channel, patch); 4 columns per lane), restructured for issue
// efficiency — the kernel is integer-issue-bound, not HBM-bound, in its naive
// form (profiles/ r1 ncu: 53 instructions per sample):
//   * row 0 peeled (no per-row "first row" test), rows >= 1 in a tight loop;
//   * the next row's 12-bit header is fetched while the current row computes;
//   * one combined validity test per row (k in 1..8 and the row fits the unit),
//     the exact error code is only worked out on the (rare) failing path;
//   * patch-edge clamping costs one select per lane per row: columns >= w of
//     a ragged patch carry "ghost" copies of column w-1, so TR of the last
//     real column is T without per-sample tests (RAGGED instantiation only);
//   * stream (G = 1) ring bookkeeping is a single compare per row; waiting,
//     refilling and the wrap mirror live on a slow path;
//   * ring reads are 2 x LDS (the second at +4, the mirror makes the wrap
//     contiguous) + 2 x PRMT + 1 funnel shift.
#pragma once

namespace l3 {

#ifndef L3_ISSUE_REL
#define L3_ISSUE_REL 1   // ring chunk issue with 32-bit A-relative bounds (the 64-bit form cost ~67 instr per chunk)
#endif
#ifndef L3_BULK_FIRST
#define L3_BULK_FIRST 0   // planar streamed tasks: the first 8 KB of a unit as one bulk copy (measured slower)
#endif
#ifndef L3_KTAB_RING
#define L3_KTAB_RING 1   // planar kernel: each warp's copy of the per-k unpack table sits after its ring
#endif
constexpr int kKtabOff = kRingBytes + 64;      // the table's offset in the warp's ring region
constexpr int kRingPitch = kRingBytes + 64 + (L3_KTAB_RING ? 256 : 0);   // ring (+ wrap mirrors) + table

__device__ __forceinline__ void st_release_gpu(unsigned int* p, unsigned int v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned int ld_acquire_gpu(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// ---------------------------------------------------------------- a7 inside the persistent launch
// a7: the last CTA to finish converts the per-image error keys (atomicMin over the units,
// key 0 = header-level error, else 1<<31 | unit<<1 | truncated) into status / bad_unit, the
// result of a sequential decode, and re-zeroes the workspace head so
// the next launch on this workspace needs no host work.
// A1: a1 ran inside the CTAs (a1_desc: this CTA's shared results, with each image's header status);
// the finisher then writes every image's status and bad_unit.
__device__ __forceinline__ void a7_finish(const ParseParams& pp, WsHead* head, unsigned int* sh_ticket,
                                          const A1Compact* a1_desc = nullptr) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    *sh_ticket = atomicAdd(&head->done_ctas, 1u);
  }
  __syncthreads();
  if (*sh_ticket != gridDim.x - 1) return;
  __threadfence();
  for (int i = threadIdx.x; i < pp.n; i += blockDim.x) {
    const uint32_t key = ~atomicExch(&pp.ws.errkey[i], 0u);   // read and re-zero (record_err encoding)
    const int32_t st = a1_desc ? a1_desc[i].st : pp.status[i];
    if (a1_desc && (st != L3_OK || key == kNoError)) {
      pp.status[i] = st;
      if (pp.bad_unit) pp.bad_unit[i] = -1;
    }
    if (st != L3_OK) continue;   // header-level error from a1
    if (key == kNoError) continue;
    if (key == 0u) {
      pp.status[i] = L3_E_CORRUPT_HEADER;
      if (a1_desc && pp.bad_unit) pp.bad_unit[i] = -1;
    } else {
      pp.status[i] = (key & 1u) ? L3_E_TRUNCATED_STREAM : L3_E_CORRUPT_STREAM;
      if (pp.bad_unit) pp.bad_unit[i] = (int32_t)((key >> 1) & 0x3FFFFFFFu);
    }
  }
  if (threadIdx.x == 0) {
    head->next_task[0] = 0;
    head->next_task[1] = 0;
    head->done_ctas = 0;
  }
}

__host__ __device__ constexpr size_t fast_smem_bytes() {
  return (size_t)kWarpsPerCta * kRingPitch + (size_t)kWarpsPerCta * kSlots * 8 + 16;
}

// 32 stream bits at unwrapped ring bit position `bit` (MSB-first, reading C8).
// Ring words are byte-swapped once when their chunk lands (swap_words), so a
// word's bit 31 is the first stream bit of that word.
// SLOTS: ring size in kSlotBytes slots (the HWC kernel runs 4-slot rings, three per warp).
template <int SLOTS = kSlots>
__device__ __forceinline__ uint32_t rbits(const uint8_t* ring, uint32_t bit) {
  const uint32_t* p =
      reinterpret_cast<const uint32_t*>(ring + ((bit >> 3) & (uint32_t)(SLOTS * kSlotBytes - 4)));
  const uint32_t hi = p[0];
  const uint32_t lo = p[1];   // at the ring end this is the mirror of word 0
  uint32_t d;
  asm("shf.l.wrap.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(lo), "r"(hi), "r"(bit));   // wraps the shift mod 32
  return d;
}

// Byte-swap the 16-byte-aligned ring bytes [lo, hi) in place (lanes stride `step` x 16 B).
__device__ __forceinline__ void swap_words(uint8_t* base, uint32_t lo, uint32_t hi, uint32_t first, uint32_t step) {
  for (uint32_t x = lo + first * 16u; x < hi; x += step * 16u) {
    uint4 v = *reinterpret_cast<uint4*>(base + x);
    v.x = bswap32(v.x);
    v.y = bswap32(v.y);
    v.z = bswap32(v.z);
    v.w = bswap32(v.w);
    *reinterpret_cast<uint4*>(base + x) = v;
  }
}

// Per-warp stream state (G == 1 tasks); warp-uniform.
struct StreamState {
  uint64_t A;           // absolute, 16-aligned start of the staged range
  uint64_t B;           // absolute, 16-aligned end of the staged range
  uint64_t stage_end;   // absolute end of the bytes that matter
  uint32_t nchunks, issued, landed;
  uint32_t landed_end;  // A-relative bytes known to be resident (0xFFFFFFFF = all)
  uint32_t group = 0;   // chunks [0, group) were issued as ONE bulk copy on bars[0] (L3_BULK_FIRST)
  // A-relative 32-bit bounds (stream_rel_init): B - A; the bytes a bulk copy may move (up to the batch end
  // rounded down to 16); stage_end - A (the lanes copy [rel_bulk, rel_end) when the unit ends past it)
  uint32_t relB, rel_bulk, rel_end;
};

template <class S>
__device__ __forceinline__ void stream_rel_init(S& s, uint64_t lim) {
  s.relB = (uint32_t)(s.B - s.A);
  s.rel_bulk = lim > s.A ? (uint32_t)(min(s.B, lim) - s.A) : 0u;
  s.rel_end = s.stage_end > s.A ? (uint32_t)(s.stage_end - s.A) : 0u;
}

// Issue chunk s.issued of [A, B) into its ring slot: one bulk copy by the leader lane (32-bit A-relative
// bounds); only a unit ending past the batch's last 16-byte boundary has lane-copied tail bytes.
template <int SLOTS, class S, int SB = kSlotBytes>
__device__ __forceinline__ void stream_issue_rel(const uint8_t* src, S& s, uint8_t* ring, uint64_t* bars, bool leader,
                                                 uint32_t lane, uint32_t lanes) {
  const uint32_t c = s.issued;
  const uint32_t ca = c * (uint32_t)SB;
  const uint32_t cb = min(ca + (uint32_t)SB, s.relB);
  const uint32_t be = min(cb, s.rel_bulk);
  const uint32_t bulk = be > ca ? be - ca : 0u;
  uint8_t* dst = ring + (c % SLOTS) * SB;
  if (leader) {
    mbar_arrive_expect_tx(&bars[c % SLOTS], bulk);
    if (bulk) bulk_g2s(dst, src + s.A + ca, bulk, &bars[c % SLOTS]);
  }
  if (s.rel_bulk < cb) {   // rare: the batch's last unit
    const uint32_t te = min(cb, s.rel_end);
    for (uint32_t x = max(ca, s.rel_bulk) + lane; x < te; x += lanes) dst[x - ca] = __ldg(src + s.A + x);
  }
  s.issued = c + 1;
}

// Wait for chunk s.landed (the first chunk of the initial group waits for the whole group).
template <int SLOTS = kSlots>
__device__ __forceinline__ void stream_land(StreamState& s, uint64_t* bars, uint32_t& phase_bits) {
  const uint32_t sl = s.landed % SLOTS;
  if (s.landed >= s.group) {
    mbar_wait(&bars[sl], (phase_bits >> sl) & 1u);
    phase_bits ^= 1u << sl;
  } else if (s.landed == 0) {
    mbar_wait(&bars[0], phase_bits & 1u);
    phase_bits ^= 1u;
  }
}

// REL: 32-bit A-relative bounds (the caller ran stream_rel_init), else the 64-bit stage_range form.
// SB: chunk (slot) bytes; the ring is SLOTS x SB bytes.
template <int SLOTS = kSlots, bool REL = (L3_ISSUE_REL != 0), int SB = kSlotBytes>
__device__ __forceinline__ void stream_issue(const uint8_t* src, uint64_t lim, StreamState& s, uint8_t* ring,
                                             uint64_t* bars, int lane) {
  if constexpr (REL) {
    stream_issue_rel<SLOTS, StreamState, SB>(src, s, ring, bars, lane == 0, (uint32_t)lane, 32u);
    return;
  }
  static_assert(REL || SB == kSlotBytes, "64-bit issue: 1 KB chunks");
  const uint32_t c = s.issued;
  const uint64_t ca = s.A + (uint64_t)c * kSlotBytes;
  const uint64_t cb = min(ca + kSlotBytes, s.B);
  stage_range(src, ca, cb, lim, s.stage_end, ring + (c % SLOTS) * kSlotBytes, &bars[c % SLOTS], lane == 0, lane,
              32);
  s.issued = c + 1;
}

// Slow path of the per-row ring test: refill consumed slots, then wait until
// `need` A-relative bytes are resident. Warp-collective.
template <int SLOTS = kSlots, bool REL = (L3_ISSUE_REL != 0), int SB = kSlotBytes>
__device__ __forceinline__ void stream_advance(const uint8_t* src, uint64_t lim, StreamState& s, uint8_t* ring,
                                            uint64_t* bars, uint32_t& phase_bits, uint32_t consumed_byte,
                                            uint32_t need, int lane) {
  const uint32_t consumed = consumed_byte / SB;
  if (s.issued < s.nchunks && s.issued < consumed + SLOTS) {
    __syncwarp();
    fence_proxy_async_smem();
    while (s.issued < s.nchunks && s.issued < consumed + SLOTS)
      stream_issue<SLOTS, REL, SB>(src, lim, s, ring, bars, lane);
    __syncwarp();
  }
  while (s.landed < s.issued && (uint64_t)s.landed * SB < need) {
    const uint32_t sl = s.landed % SLOTS;
    stream_land<SLOTS>(s, bars, phase_bits);
    __syncwarp();
    swap_words(ring, sl * SB, (sl + 1) * SB, lane, 32);
    __syncwarp();
    if (sl == 0) {   // keep the 16-byte mirror of word 0.. after the ring end current
      if (lane < 4)
        reinterpret_cast<uint32_t*>(ring + SLOTS * SB)[lane] = reinterpret_cast<uint32_t*>(ring)[lane];
      __syncwarp();
    }
    s.landed++;
  }
  s.landed_end = (s.landed == s.nchunks) ? 0xFFFFFFFFu : s.landed * SB;
}

#ifndef L3_STREAM_SB
#define L3_STREAM_SB 1024   // fp32 planar streamed path: chunk bytes of the 8 KB ring (2048: 4 chunks)
#endif
template <bool F32> __host__ __device__ constexpr int kStreamSB() { return F32 ? L3_STREAM_SB : kSlotBytes; }
template <bool F32> __host__ __device__ constexpr int kStreamSlots() { return kRingBytes / kStreamSB<F32>(); }

// ---------------------------------------------------------------- SWAR core
// Two samples per 32-bit register, one per 16-bit half (value in the half's
// low byte, high byte zero): "pair" form. Only native sm_100a SIMD ops are
// used (VABSDIFF4.U8, VIMNMX.U16x2, VIMNMX3.U16x2, PRMT); the key arithmetic
// runs on the FMA pipe (IMAD), relieving the half-rate ALU pipe that bounds
// the scalar form (profiles/: ALU pipe 78% busy).

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t d;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
  return d;
}
__device__ __forceinline__ uint32_t shr_c(uint32_t x, uint32_t n) {   // clamped shift (PTX semantics)
  uint32_t d;
  asm("shr.b32 %0, %1, %2;" : "=r"(d) : "r"(x), "r"(n));
  return d;
}
__device__ __forceinline__ uint32_t shl_c(uint32_t x, uint32_t n) {
  uint32_t d;
  asm("shl.b32 %0, %1, %2;" : "=r"(d) : "r"(x), "r"(n));
  return d;
}

// Custom Paeth predictor (Fig. 3; ties TL, T, TR — reading C3)
// for two samples in pair form. With u = |TL-T|, v = |TR-T|, w = |TL-TR| the
// distances to ref = TL+TR-T are d(TL) = v, d(T) = |TL+TR-2T| = 2max(u,v) - w,
// d(TR) = u. Adding w to all three keeps the order and makes the
// keys non-negative: k = (dist + w) << 7 | c, where the low bits c encode both
// the tie rank and the byte index of that candidate in {X = [TL0,T0,TL1,T1],
// Y = [TR0,0,TR1,0]}, so the minimum key's low nibbles are directly the PRMT
// selector of the winner (keys <= 510 << 7 | 6 fit 16 bits).
__device__ __forceinline__ uint32_t paeth_pred2(uint32_t tl, uint32_t t, uint32_t tr, uint32_t K) {
  const uint32_t u = __vabsdiffu4(tl, t);
  const uint32_t v = __vabsdiffu4(tr, t);
  const uint32_t w = __vabsdiffu4(tl, tr);
  const uint32_t mx = __vmaxu2(u, v);
  // K = 128 arrives as a runtime value so the key arithmetic stays on IMAD
  // (FMA pipe) instead of LEA (ALU pipe). Low 7 bits: 0x50 | byte index; the 5
  // in bits 4-6 makes the unused PRMT nibbles (1 and 3) pick byte 5 = 0 (or its
  // sign, also 0), so the result's bytes 1 and 3 are zero.
  const uint32_t kTL = v * K + (w * K + 0x00520050u);   // candidate bytes: s0 -> 0, s1 -> 2
  const uint32_t kTR = u * K + (w * K + 0x00560054u);   // s0 -> 4, s1 -> 6
  const uint32_t kT = mx * (2u * K) + 0x00530051u;      // s0 -> 1, s1 -> 3
  const uint32_t m = __vimin3_u16x2(kTL, kT, kTR);
  const uint32_t X = prmt(tl, t, 0x6240);
  const uint32_t sel = prmt(m, 0, 0x4420);   // nibble0 <- half0 code, nibble2 <- half1 code
  return prmt(X, tr, sel);                   // pair form: bytes 1 and 3 are zero
}

// Custom Paeth predictor (Fig. 3; ties TL, T, TR — reading C3) for two samples held as
// BIASED HALVES: each 16-bit half is the fp16 value 1024 + c (bits 0x6400 | c), so differences are exact
// small integers and the bits stay an integer pair for the mod-256 residual add. With a = TL - T,
// b = TR - T, s = a + b the distances are d(TL) = |b|, d(T) = |s|, d(TR) = |a|, and for
// integers sat(x - y) = [x > y]. TL wins iff |b| <= min(|a|, |s|), i.e. x1 = sat(|b| - min(|a|, |s|)) = 0;
// TR wins iff |a| < min(|b|, |s|), i.e. r = sat(min(|b|, |s|) - |a|) = 1; else T. So
// pred = (TL - a·x1) + b·r: x1 = 0 gives TL, x1 = 1 gives T, plus b when TR wins (then x1 = 1). That is
// 7 HADD2 / HFMA2 on the FMA pipes and 2 HMNMX2 on the ALU (|x| and .SAT fold into the instructions).
// Every intermediate is an integer of magnitude <= 1534 (exact in fp16). DESIGN.md §5;
// exhaustively checked by l3_selftest_paeth_h2.
__device__ __forceinline__ __half2 u2h2(uint32_t u) { return *reinterpret_cast<__half2*>(&u); }
__device__ __forceinline__ uint32_t h22u(__half2 h) { return *reinterpret_cast<uint32_t*>(&h); }
#ifndef L3_H2_MIN
#define L3_H2_MIN 1   // 1: the 9-op form with two HMNMX2; 0: the 11-op all-FMA-pipe form
#endif
__device__ __forceinline__ uint32_t paeth_h2(uint32_t tl, uint32_t t, uint32_t tr) {
  const __half2 TL = u2h2(tl), T = u2h2(t), TR = u2h2(tr);
  const __half2 a = __hsub2(TL, T), b = __hsub2(TR, T), s = __hadd2(a, b);
  const __half2 A = __habs2(a), B = __habs2(b), S = __habs2(s);
#if L3_H2_MIN
  const __half2 x1 = __hsub2_sat(B, __hmin2(A, S));   // [TL does not win]
  const __half2 r = __hsub2_sat(__hmin2(B, S), A);    // [TR wins]
  return h22u(__hfma2(b, r, __hfma2(a, __hneg2(x1), TL)));
#else
  const __half2 q = __hsub2_sat(B, A);    // [|b| > |a|]
  const __half2 r1 = __hsub2_sat(B, S);   // [|b| > |s|]
  const __half2 r2 = __hsub2_sat(S, A);   // [|s| > |a|]
  const __half2 u1 = __hsub2(__float2half2_rn(1.f), q);
  const __half2 itl = __hfma2(u1, __hneg2(r1), u1);   // (1 - q)(1 - r1)
  const __half2 itr = __hmul2(q, r2);
  return h22u(__hfma2(b, itr, __hfma2(a, itl, T)));
#endif
}

#ifndef L3_BIAS_LOP3
#define L3_BIAS_LOP3 1
#endif
__device__ __forceinline__ uint32_t bias_reg(uint32_t K) { return K * 0x00C800C8u; }
__device__ __forceinline__ uint32_t lo_bytes_biased(uint32_t x, uint32_t bias) {
#if L3_BIAS_LOP3
  uint32_t d;
  asm("lop3.b32 %0, %1, 0x00FF00FF, %2, 0xEA;" : "=r"(d) : "r"(x), "r"(bias));   // (a & b) | c
  return d;
#else
  return (x & 0x00FF00FFu) | 0x64006400u;
#endif
}

#ifndef L3_H2_F32
#define L3_H2_F32 0xF   // fp32 planar / crop paths
#endif
#ifndef L3_H2_U8
#define L3_H2_U8 0xF    // u8 planar / crop paths (0: the byte-form paeth_pred4)
#endif
#ifndef L3_H2_WIDE
#define L3_H2_WIDE 0xF  // u8 wide 8-column path: bit i = pair i of the lane's 4 pairs runs paeth_h2 (C4 -1.6 % vs 0x5)
#endif
#ifndef L3_REFILL_AHEAD
#define L3_REFILL_AHEAD 2048   // streamed ring: land 2 KB beyond the next two rows per refill call (fewer calls)
#endif
#ifndef L3_UNPACK_TAB
#define L3_UNPACK_TAB 1   // delta unpack by shift amounts / mask from a per-k shared table (C3 u8 -2.5 %, fp32 -1.2 %)
#endif
// Per-k unpack table (L3_UNPACK_TAB): {32 - k, 16 - 2k, 2k, ((1 << k) - 1) << 16} for k = 1..8, zeros for the
// invalid k (their rows are flagged by the validity accumulator). Every kernel that runs decode_row fills it.
__shared__ uint4 l3_ktab[16];
// Table entry k by a 32-bit shared-window address (ld.shared): the generic-pointer form made ptxas
// rebuild the entry's cluster-window address (S2R SR_CgaCtaId + 3 ops) in every row.
__device__ __forceinline__ uint4 ktab_entry(uint32_t k) {
  uint4 v;
  asm("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
      : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
      : "r"((uint32_t)__cvta_generic_to_shared(l3_ktab) + 16u * k));
  return v;
}
__device__ __forceinline__ void init_ktab() {
  if (threadIdx.x < 16) {
    const uint32_t k = threadIdx.x;
    l3_ktab[k] = (k >= 1 && k <= 8) ? make_uint4(32u - k, 16u - 2u * k, 2u * k, ((1u << k) - 1u) << 16)
                                    : make_uint4(0u, 0u, 0u, 0u);
  }
}
#ifndef L3_UNPACK_SHF
#define L3_UNPACK_SHF 1   // fp32 delta unpack: 0 = left shifts as IMAD, 1 = as SHF (u8 paths keep IMAD)
#endif
#ifndef L3_H2_HWC
#define L3_H2_HWC 0xF   // HWC tile kernel (rows left in s.A / s.B for the interleaving store): C3 HWC -7 %
#endif
#ifndef L3_H2_CVT
#define L3_H2_CVT 0     // fp32 stores of biased halves: 1 = HADD2 + HADD2.F32 (FMA pipes), 0 = I2F.U8 (XU)
#endif

#ifndef L3_U8_V16
#define L3_U8_V16 0   // A/B: u8 rows as 128-bit stores (4-lane shuffle gather) where aligned; measured slower
#endif
#ifndef L3_MIN_CTAS
#define L3_MIN_CTAS 6   // __launch_bounds__ min CTAs per SM for the planar kernels: register cap 80, no spills
#endif
#ifndef L3_CROP_MIN_CTAS
#define L3_CROP_MIN_CTAS 0   // crop (f3) kernels: no register cap (96 registers, 5 CTAs per SM)
#endif
#ifndef L3_SMEM_PREFIX
#define L3_SMEM_PREFIX 1   // per-CTA shared-memory copy of the task prefix for the image lookup (n <= 256)
#endif
constexpr int kShPrefix = 256;
#ifndef L3_EDGE_SEL
#define L3_EDGE_SEL 0   // 1: patch-edge clamps by per-lane PRMT selectors instead of selects (A/B option)
#endif
#ifndef L3_PRED4
#define L3_PRED4 1   // byte-form 4-sample predictor on the u8 storing paths
#endif

// Custom Paeth predictor (Fig. 3; ties TL, T, TR — reading C3)
// for the lane's 4 samples in byte form. The candidates of sample i are
// c[i-1], c[i], c[i+1] of the previous row; L = [c-1 c0 c1 c2], Q = [c0 c1 c2 c3],
// R = [c1 c2 c3 c4] (edge-clamped by the caller's selectors). With u = |TL-T|,
// v = |TR-T|, w = |TL-TR| the distances to ref = TL+TR-T are d(TL) = v, d(TR) = u and
// d(T) = |TL+TR-2T|, which is |u-v| when T lies between TL and TR (then w = u+v) and
// u+v >= max(u,v) when it does not (then w = |u-v|, and T can never be the
// strict minimum, so its distance may be replaced by 255). So the per-sample
// distances fit a byte: keys are dist << 8 | code in 16x2 halves (samples 0,2 in
// pair A, 1,3 in pair B), one VIMNMX3.U16x2 per pair picks min distance, ties by
// code order TL < T < TR, and the winning codes are directly the nibbles of a
// PRMT selector into (L, R) bytes: sample i's candidates live at L/R byte indices
// {0,1,2}, {1,2,3}, {2,3,6}, {3,6,7} for i = 0..3 (monotone in tie rank).
// DESIGN.md §5 (byte-form predictor); exhaustively checked by l3_selftest_paeth4.
__device__ __forceinline__ uint32_t paeth_pred4(uint32_t L, uint32_t Q, uint32_t R) {
  const uint32_t U = __vabsdiffu4(L, Q);   // u_i = d(TR)
  const uint32_t V = __vabsdiffu4(R, Q);   // v_i = d(TL)
  const uint32_t W = __vabsdiffu4(L, R);   // w_i
  const uint32_t D = __vabsdiffu4(U, V);   // |u - v|
  // bytes with W == D (T not strictly between TL and TR): force d(T) = 255
  const uint32_t a = (W ^ D) & 0x7F7F7F7Fu;
  const uint32_t b = a + 0x7F7F7F7Fu;       // bit 7 set iff the low 7 bits of W^D are non-zero
  const uint32_t c = ~(b | (W ^ D));        // bit 7 of byte i set iff W_i == D_i
  const uint32_t Dm = D | prmt(c, 0u, 0xBA98u);   // sign-replicate bit 7 of each byte
  // keys: byte 1 / 3 of each half = distance, byte 0 / 2 = code (PRMT from the code words)
  constexpr uint32_t kCodeTL = 0x30021000u, kCodeT = 0x60032001u, kCodeTR = 0x70063002u;
  const uint32_t mA = __vimin3_u16x2(prmt(V, kCodeTL, 0x2604u), prmt(Dm, kCodeT, 0x2604u), prmt(U, kCodeTR, 0x2604u));
  const uint32_t mB = __vimin3_u16x2(prmt(V, kCodeTL, 0x3715u), prmt(Dm, kCodeT, 0x3715u), prmt(U, kCodeTR, 0x3715u));
  const uint32_t t = mA | mB;               // byte 0: code0 | code1 << 4, byte 2: code2 | code3 << 4
  return prmt(L, R, prmt(t, 0u, 0x0020u));
}

// Row reconstruction state of one lane: 4 consecutive columns j4..j4+3.
struct LaneRows {
  uint32_t bp;        // unwrapped ring bit position of the current row header
  uint32_t lim;       // bit limit of the unit (same origin as bp)
  uint32_t w;         // unit width
  uint32_t h;         // unit height (0: inactive lane)
  uint32_t j4;        // first column of this lane
  uint32_t raw;       // the 32 stream bits starting at the current row header
  uint32_t kacc;      // max over rows of (raw - 2^28): >= 2^31 iff some k was 0 or > 8
  bool first, last, valid;
  uint8_t* optr;      // output of column j4 in the current row
  uint32_t pitch;     // bytes between output rows
  uint32_t A, B;      // previous row, pair form: A = (c0, c1), B = (c2, c3) (pair-predictor paths)
  uint32_t Q;         // previous row, byte form [c0 c1 c2 c3] (byte-predictor paths)
  uint32_t selL;      // PRMT selector (left lane's Q, Q) -> [c-1 c0 c1 c2], clamped at column 0
  uint32_t selR;      // PRMT selector (Q, right lane's Q) -> [c1 c2 c3 c4], clamped at the last lane
  uint32_t selG;      // RAGGED: PRMT selector replicating column w-1 into the lane's ghost columns
  bool v16;           // u8 FAST: 16-byte rows (every 4 lanes' words gathered into one 128-bit store)
  // CROP variant only (f3, partial decode): output window mapping
  int32_t ri;         // current image row - crop top
  uint32_t chh;       // crop height
  uint32_t cmask;     // which of the lane's 4 output elements are inside the patch and the window
  uint32_t qsel;      // PRMT selector putting the lane's samples in output order (flip: reversed)
};

// FAST: aligned vector store. Otherwise scalar stores; RAGGED: the patch width is not a multiple of
// 4, so the lane's trailing columns may lie outside it (else all 4 are stored unconditionally).
// H2: biased-half pairs (0x6400 | c per half): c = (1024 + c) - 1024 by one HADD2 per pair, then the
// fp16 -> fp32 conversion (HADD2.F32) and the normalise FFMA, all off the ALU pipe.
template <bool F32, bool FAST, bool RAGGED = !FAST, bool H2 = false>
__device__ __forceinline__ void store4(const LaneRows& s, uint32_t xA, uint32_t xB, float sc, float bi, bool pred) {
  if (F32) {
    float c0, c1, c2, c3;
    if (H2 && L3_H2_CVT) {
      const float2 fa = __half22float2(__hsub2(u2h2(xA), __float2half2_rn(1024.f)));
      const float2 fb = __half22float2(__hsub2(u2h2(xB), __float2half2_rn(1024.f)));
      c0 = fa.x; c1 = fa.y; c2 = fb.x; c3 = fb.y;
    } else if (H2) {
      c0 = (float)(xA & 0xFFu); c1 = (float)((xA >> 16) & 0xFFu); c2 = (float)(xB & 0xFFu); c3 = (float)((xB >> 16) & 0xFFu);
    } else {
      c0 = (float)(xA & 0xFFFFu); c1 = (float)(xA >> 16); c2 = (float)(xB & 0xFFFFu); c3 = (float)(xB >> 16);
    }
    const float v0 = fmaf(c0, sc, bi), v1 = fmaf(c1, sc, bi);
    const float v2 = fmaf(c2, sc, bi), v3 = fmaf(c3, sc, bi);
    if (FAST) {   // predicated STG.128, no branch
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %5, 0;\n\t"
          "@p st.global.v4.f32 [%0], {%1, %2, %3, %4};\n\t}" ::"l"(s.optr),
          "f"(v0), "f"(v1), "f"(v2), "f"(v3), "r"((uint32_t)pred));
    } else if (pred) {
      float* o = reinterpret_cast<float*>(s.optr);
      o[0] = v0;
      if (!RAGGED || s.j4 + 1 < s.w) o[1] = v1;
      if (!RAGGED || s.j4 + 2 < s.w) o[2] = v2;
      if (!RAGGED || s.j4 + 3 < s.w) o[3] = v3;
    }
  } else {
    const uint32_t q = prmt(xA, xB, 0x6420);   // [c0, c1, c2, c3]
    if (FAST) {
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %2, 0;\n\t"
          "@p st.global.b32 [%0], %1;\n\t}" ::"l"(s.optr), "r"(q), "r"((uint32_t)pred));
    } else if (pred) {
      uint8_t* o = s.optr;
      o[0] = (uint8_t)q;
      if (!RAGGED || s.j4 + 1 < s.w) o[1] = (uint8_t)(q >> 8);
      if (!RAGGED || s.j4 + 2 < s.w) o[2] = (uint8_t)(q >> 16);
      if (!RAGGED || s.j4 + 3 < s.w) o[3] = (uint8_t)(q >> 24);
    }
  }
}

// Byte-form variant of store4: q = [c0 c1 c2 c3].
template <bool F32, bool FAST, bool RAGGED = !FAST>
__device__ __forceinline__ void store4q(const LaneRows& s, uint32_t q, float sc, float bi, bool pred, uint32_t Lw) {
  if (F32) {
    const float v0 = fmaf((float)(q & 0xFFu), sc, bi), v1 = fmaf((float)((q >> 8) & 0xFFu), sc, bi);
    const float v2 = fmaf((float)((q >> 16) & 0xFFu), sc, bi), v3 = fmaf((float)(q >> 24), sc, bi);
    if (FAST) {   // predicated STG.128, no branch
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %5, 0;\n\t"
          "@p st.global.v4.f32 [%0], {%1, %2, %3, %4};\n\t}" ::"l"(s.optr),
          "f"(v0), "f"(v1), "f"(v2), "f"(v3), "r"((uint32_t)pred));
    } else if (pred) {
      float* o = reinterpret_cast<float*>(s.optr);
      o[0] = v0;
      if (!RAGGED || s.j4 + 1 < s.w) o[1] = v1;
      if (!RAGGED || s.j4 + 2 < s.w) o[2] = v2;
      if (!RAGGED || s.j4 + 3 < s.w) o[3] = v3;
    }
  } else {
    if (FAST && s.v16) {   // 128-bit stores: lane 4m gathers lanes 4m+1..4m+3's words (warp-uniform branch)
      const uint32_t q1 = __shfl_down_sync(0xffffffffu, q, 1, Lw);
      const uint32_t q2 = __shfl_down_sync(0xffffffffu, q, 2, Lw);
      const uint32_t q3 = __shfl_down_sync(0xffffffffu, q, 3, Lw);
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %5, 0;\n\t"
          "@p st.global.v4.b32 [%0], {%1, %2, %3, %4};\n\t}" ::"l"(s.optr),
          "r"(q), "r"(q1), "r"(q2), "r"(q3), "r"((uint32_t)(pred && (s.j4 & 15u) == 0)));
    } else if (FAST) {
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %2, 0;\n\t"
          "@p st.global.b32 [%0], %1;\n\t}" ::"l"(s.optr), "r"(q), "r"((uint32_t)pred));
    } else if (pred) {
      uint8_t* o = s.optr;
      o[0] = (uint8_t)q;
      if (!RAGGED || s.j4 + 1 < s.w) o[1] = (uint8_t)(q >> 8);
      if (!RAGGED || s.j4 + 2 < s.w) o[2] = (uint8_t)(q >> 16);
      if (!RAGGED || s.j4 + 3 < s.w) o[3] = (uint8_t)(q >> 24);
    }
  }
}

// f3: store the lane's 4 samples into a cropped (optionally flipped) window, planar or HWC. s.optr
// walks the output row by row at the lane's lowest-address element (flip: the lane's 4 samples are
// reversed into output order by the s.qsel PRMT), so the 4 elements sit at fixed immediate offsets;
// s.cmask holds which of them are inside the patch and the window (fixed per task). Pair form
// (xA, xB), or (BYTES) byte form [c0 c1 c2 c3] in xA.
template <bool F32, bool HWC, bool BYTES = false>
__device__ __forceinline__ void store4_crop(const LaneRows& s, uint32_t xA, uint32_t xB, float sc, float bi,
                                            bool live) {
  constexpr uint32_t kStep = (HWC ? 3u : 1u) * (F32 ? 4u : 1u);   // bytes between the lane's elements
  const bool rowok = live && (uint32_t)s.ri < s.chh;
  const uint32_t qq = prmt(BYTES ? xA : prmt(xA, xB, 0x6420u), 0u, s.qsel);
#pragma unroll
  for (int t = 0; t < 4; t++) {
    if (rowok && ((s.cmask >> t) & 1u)) {
      const uint32_t x = (qq >> (8 * t)) & 0xFFu;
      if (F32) *reinterpret_cast<float*>(s.optr + t * kStep) = fmaf((float)x, sc, bi);
      else s.optr[t * kStep] = (uint8_t)x;
    }
  }
}

// One row of one lane (a3-a6). FIRST: row 0 of the patch (no prediction,
// PAPER.md:139 "the first row is stored in a raw data format").
// Validity is accumulated, not tested per row: kacc collects every row's k
// (a k outside 1..8 sets its top bit) and a row overrunning the unit leaves
// bp > lim after the patch (bp only grows). Decoding continues on garbage in
// that case (reads stay inside the ring, writes inside the patch) and the
// exact first error is re-derived after the patch (unit_first_error).
// GUARD: rows may run past this lane's h (G > 1 segments of unequal height).
// STORE = false (HWC kernel): the row's pixels are left in s.A / s.B for an interleaving store.
// KT: 0 = the per-k table in the static shared array; else its byte offset from `ring` (the planar
// kernel's per-warp copy, addressed from the ring's base register: no per-row address rebuild).
template <bool FIRST, bool F32, bool FAST, bool GUARD, bool CROP, bool STORE = true, int SLOTS = kSlots,
          bool HWC = false, bool RAGGED = !FAST, int PAR = 0, int KT = 0>
__device__ __forceinline__ void decode_row(LaneRows& s, const uint8_t* ring, uint32_t r, uint32_t Lw_rt, float sc,
                                           float bi, uint32_t K) {
  const uint32_t Lw = GUARD ? Lw_rt : 32u;   // stream (G == 1) tasks span the whole warp
  // a3: row header (PAPER.md:152 step 1): 4-bit k, 8-bit base
  const uint32_t k = s.raw >> 28;
  const uint32_t base2 = (s.raw >> 20) * 0x00010001u;   // (k:4 | base:8) per half; k bits masked below
  const uint32_t rowbits = 12u + k * s.w;
  const bool live = GUARD ? (r < s.h) : true;
  const uint32_t nbp = s.bp + rowbits;
  const uint32_t raw_next = rbits<SLOTS>(ring, nbp);    // next row's header, fetched early
  // a4: pixel-wise delta unpack (PAPER.md:152 step 2, :187): field = 4 k-bit deltas, MSB-first
  const uint32_t field = rbits<SLOTS>(ring, s.bp + 12u + s.j4 * k);
#if L3_UNPACK_TAB
  // the row's shift amounts and mask from the per-k table (one broadcast LDS.128, issued beside the
  // field's loads): dA = (d1 << 16) | d0 from field >> (16 - 2k) (d1 lands at bit 16) and
  // field >> (32 - k); dB the same from field << 2k
  const uint4 T = KT ? *reinterpret_cast<const uint4*>(ring + KT + 16u * k) : ktab_entry(k);
  const uint32_t g = shl_c(field, T.z);
  const uint32_t dA = ((shr_c(field, T.y) & T.w) | shr_c(field, T.x)) + base2;
  const uint32_t dB = ((shr_c(g, T.y) & T.w) | shr_c(g, T.x)) + base2;
#else
  const uint32_t sh = 32u - k;
  const uint32_t d0 = shr_c(field, sh);
  uint32_t d1, d2, d3;
#if L3_UNPACK_SHF
  if (F32) {   // the left shifts on the ALU pipe (balances the FMA-pipe-heavy fp32 predictor mix)
  d1 = shr_c(shl_c(field, k), sh);
  d2 = shr_c(shl_c(field, 2u * k), sh);
  d3 = shr_c(shl_c(field, 3u * k), sh);
  } else
#endif
  {             // the left shifts as multiplies (IMAD, FMA pipe)
  const uint32_t pk = shl_c(1u, k);
  d1 = shr_c(field * pk, sh);
  d2 = shr_c(field * (pk * pk), sh);
  d3 = shr_c(field * (pk * pk * pk), sh);
  }
  const uint32_t dA = d1 * 0x10000u + d0 + base2;
  const uint32_t dB = d3 * 0x10000u + d2 + base2;
#endif
  // byte-form predictor: u8 planar / crop stores (measured: C2 -1.7 %, C3 u8 neutral, fp32 +5 %)
  constexpr bool P4 = STORE && !F32 && (L3_PRED4 != 0) && (L3_H2_U8 == 0);
  // biased-half pair form (paeth_h2): halves hold 0x6400 | c instead of c
  constexpr int kH2Mask = STORE ? (F32 ? L3_H2_F32 : L3_H2_U8) : L3_H2_HWC;
  constexpr bool H2 = kH2Mask != 0;
  constexpr int HM = (kH2Mask >> (2 * PAR)) & 3;
  uint32_t xA, xB;
  if (P4) {
    if (FIRST) {
      xA = dA;
      xB = dB;
    } else {
      // a5: row-wise parallel custom Paeth, 4 samples in byte form
      const uint32_t Lq = __shfl_up_sync(0xffffffffu, s.Q, 1, Lw);     // left lane's [c-4 .. c-1]
      const uint32_t Rq = __shfl_down_sync(0xffffffffu, s.Q, 1, Lw);   // right lane's [c4 .. c7]
      const uint32_t L = prmt(Lq, s.Q, s.selL);   // [c-1 c0 c1 c2]; column 0: c-1 := c0 (reading C4)
      const uint32_t R = prmt(s.Q, Rq, s.selR);   // [c1 c2 c3 c4]; last lane: c4 := c3 (C4; ghosts when ragged)
      const uint32_t pr = paeth_pred4(L, s.Q, R);
      xA = prmt(pr, 0u, 0x4140u) + dA;   // pair form (c0, c1) + residual; carries land in bytes 1, 3
      xB = prmt(pr, 0u, 0x4342u) + dB;
    }
    uint32_t q = prmt(xA, xB, 0x6420u);   // [c0 c1 c2 c3] mod 256
    if (RAGGED) q = prmt(q, 0u, s.selG);  // columns >= w: ghosts of column w-1
    if (CROP) store4_crop<F32, HWC, true>(s, q, 0u, sc, bi, live);
    else store4q<F32, FAST, RAGGED>(s, q, sc, bi, live && s.valid, Lw);
    s.Q = q;
  } else {
  if (FIRST) {
    xA = H2 ? lo_bytes_biased(dA, bias_reg(K)) : (dA & 0x00FF00FFu);
    xB = H2 ? lo_bytes_biased(dB, bias_reg(K)) : (dB & 0x00FF00FFu);
  } else {
    // a5: row-wise parallel custom Paeth
    const uint32_t Bl = __shfl_up_sync(0xffffffffu, s.B, 1, Lw);     // left lane's (c2, c3)
    const uint32_t Ar = __shfl_down_sync(0xffffffffu, s.A, 1, Lw);   // right lane's (c0, c1)
#if L3_EDGE_SEL
    // edge clamps folded into per-lane PRMT selectors (no select per row)
    const uint32_t TLA = prmt(Bl, s.A, s.selL);       // (c-1, c0); column 0: (c0, c0) (C4)
    const uint32_t TRA = prmt(s.A, s.B, 0x5412);      // (c1, c2) = TL of pair B
    const uint32_t TRB = prmt(s.B, Ar, s.selR);       // (c3, c+4); last lane: (c3, c3) (C4; ghosts when ragged)
#else
    const uint32_t LF = s.first ? (s.A << 16) : Bl;   // byte 2 = TL of column j4 (C4: T at column 0)
    const uint32_t RT = s.last ? (s.B >> 16) : Ar;    // byte 0 = TR of column j4+3 (C4; ghosts when ragged)
    const uint32_t TLA = prmt(LF, s.A, 0x5452);       // (c-1, c0)
    const uint32_t TRA = prmt(s.A, s.B, 0x5412);      // (c1, c2) = TL of pair B
    const uint32_t TRB = prmt(s.B, RT, 0x5412);       // (c3, c+4)
#endif
    if (H2) {   // (0x6400 | pred) + residual + (k:4 | base:8): keep the low byte, restore the bias
      const uint32_t pA = (HM & 1) ? paeth_h2(TLA, s.A, TRA) : paeth_pred2(TLA, s.A, TRA, K);
      const uint32_t pB = (HM & 2) ? paeth_h2(TRA, s.B, TRB) : paeth_pred2(TRA, s.B, TRB, K);
      xA = lo_bytes_biased(pA + dA, bias_reg(K));
      xB = lo_bytes_biased(pB + dB, bias_reg(K));
    } else {
      xA = (paeth_pred2(TLA, s.A, TRA, K) + dA) & 0x00FF00FFu;
      xB = (paeth_pred2(TRA, s.B, TRB, K) + dB) & 0x00FF00FFu;
    }
  }
  if (RAGGED) {   // ragged patch: columns >= w are ghosts of column w-1
    if (s.j4 + 1 >= s.w) xA = (xA & 0xFFFFu) * 0x00010001u;
    if (s.j4 + 2 >= s.w) xB = (xA >> 16) * 0x00010001u;
    if (s.j4 + 3 >= s.w) xB = (xB & 0xFFFFu) * 0x00010001u;
  }
  // a6: store (u8 planar, or fused cast + normalise)
  if (!STORE) {
  } else if (CROP) {
    store4_crop<F32, HWC>(s, xA, xB, sc, bi, live);
  } else {
    store4<F32, FAST, RAGGED, H2>(s, xA, xB, sc, bi, live && s.valid);
  }
  s.A = xA;
  s.B = xB;
  }
  if (live) {
    s.kacc = max(s.kacc, s.raw - 0x10000000u);
    s.bp = nbp;
    s.raw = raw_next;
  }
  if (!STORE) {
  } else if (CROP) {
    s.ri++;
    s.optr += s.pitch;
  } else {
    s.optr += s.pitch;
  }
}

template <bool F32, bool FAST, bool STREAM, bool CROP, bool HWC, bool RAGGED = !FAST>
__device__ __forceinline__ void decode_unit_rows(LaneRows& s, uint8_t* ring, uint32_t hmax, uint32_t Lw, float sc,
                                                 float bi, uint32_t K, const uint8_t* src, uint64_t lim,
                                                 StreamState& st, uint64_t* bars, uint32_t& phase_bits,
                                                 uint32_t rowmax, int lane) {
  constexpr bool GUARD = !STREAM;   // G == 1: every lane runs exactly the unit's h rows
  // 32-bit chunk issue on the fp32 kernel only: the u8 narrow kernel measured slower with it (codegen)
  if (STREAM && (s.bp >> 3) + 2u * rowmax > st.landed_end)
    stream_advance<kStreamSlots<F32>(), F32 && L3_ISSUE_REL != 0, kStreamSB<F32>()>(src, lim, st, ring, bars, phase_bits, s.bp >> 3,
                                                      (s.bp >> 3) + 2u * rowmax + L3_REFILL_AHEAD, lane);
  s.raw = rbits(ring, s.bp);
  constexpr int KT = L3_KTAB_RING ? kKtabOff : 0;
  decode_row<true, F32, FAST, GUARD, CROP, true, kSlots, HWC, RAGGED, 0, KT>(s, ring, 0, Lw, sc, bi, K);
  uint32_t r = 1;
  for (; r + 1 < hmax; r += 2) {   // two rows per ring test
    if (STREAM && (s.bp >> 3) + 2u * rowmax > st.landed_end)
      stream_advance<kStreamSlots<F32>(), F32 && L3_ISSUE_REL != 0, kStreamSB<F32>()>(src, lim, st, ring, bars, phase_bits, s.bp >> 3,
                                                        (s.bp >> 3) + 2u * rowmax + L3_REFILL_AHEAD, lane);
    decode_row<false, F32, FAST, GUARD, CROP, true, kSlots, HWC, RAGGED, 0, KT>(s, ring, r, Lw, sc, bi, K);
    decode_row<false, F32, FAST, GUARD, CROP, true, kSlots, HWC, RAGGED, 1, KT>(s, ring, r + 1, Lw, sc, bi, K);
  }
  if (r < hmax) {
    if (STREAM && (s.bp >> 3) + rowmax > st.landed_end)
      stream_advance<kStreamSlots<F32>(), F32 && L3_ISSUE_REL != 0, kStreamSB<F32>()>(src, lim, st, ring, bars, phase_bits, s.bp >> 3,
                                                        (s.bp >> 3) + rowmax, lane);
    decode_row<false, F32, FAST, GUARD, CROP, true, kSlots, HWC, RAGGED, 0, KT>(s, ring, r, Lw, sc, bi, K);
  }
}

// Exact first error of a unit whose row loop raised `err`, re-derived from the
// compressed bytes in global memory with the sequential rules of a3/a7
// (k = 0 or k > 8 -> CORRUPT_STREAM; too few bits -> TRUNCATED).
__device__ __noinline__ int unit_first_error(const uint8_t* src, uint64_t start, uint64_t end, uint32_t w,
                                             uint32_t h) {
  const uint64_t len_bits = (end - start) * 8ull;
  uint64_t pos = 0;
  for (uint32_t r = 0; r < h; r++) {
    if (len_bits - pos < 4) return L3_E_TRUNCATED_STREAM;
    const uint64_t byte = start + (pos >> 3);
    const uint32_t two = ((uint32_t)src[byte] << 8) | (byte + 1 < end ? (uint32_t)src[byte + 1] : 0u);
    const uint32_t k = (two >> (12 - (pos & 7))) & 0xFu;
    if (k == 0 || k > 8) return L3_E_CORRUPT_STREAM;
    if (len_bits - pos < 12ull + (uint64_t)k * w) return L3_E_TRUNCATED_STREAM;
    pos += 12ull + (uint64_t)k * w;
  }
  return L3_OK;
}

}  // namespace l3

#include "l3_decode_wide8.cuh"

namespace l3 {

// Variants (measured): without the wide 8-column path the kernel
// fits 80 registers = 6 CTAs / 24 warps per SM (fp32 out, and u8 batches of
// small patches); WIDE (u8 out, L3_DECODE_HINT_WIDE) carries the 8-column path
// for 33 <= N <= 128 and runs at 4 CTAs per SM.
// HWC (with CROP only): the augment variant writes the window interleaved [h, w, 3].
// a1 inside a decode CTA (n <= kA1InMaxN = 32, warp 0): the same header parse and decomposition as
// l3_prep_kernel's, kept in this CTA's shared memory: compact descriptors and the
// exclusive task prefixes of the two classes (N <= 128, N > 128), totals at [n].
// WIDE: the wide kernel's decomposition (parse_phase): images whose class-0 units start within the
// batch's last tail_units units run as 1-patch tasks (the tail zone), the others keep the 8-column modes.
template <bool WIDE>
__device__ __forceinline__ void a1_in_cta(const ParseParams& pp, int lane, uint32_t* pre0, uint32_t* pre1,
                                          A1Compact* a1d) {
  uint32_t t0 = 0, t1 = 0;
  ImgDesc d;
  int st = L3_E_INVALID_ARGUMENT;
  uint64_t units = 0;
  if (lane < pp.n) {
    st = parse_header<false, false>(pp, lane, d);
    if (st == L3_OK && d.mode != 3) units = 3ull * d.P;
  }
  uint64_t uex = 0, total_units = 0;
  if (WIDE) {   // exclusive scan of the class-0 units over the batch
    uint64_t iu = units;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t v = __shfl_up_sync(0xffffffffu, iu, o);
      if (lane >= o) iu += v;
    }
    uex = iu - units;
    total_units = __shfl_sync(0xffffffffu, iu, 31);
  }
  if (lane < pp.n) {
    A1Compact c = {};
    c.st = st;
    if (st == L3_OK) {
      if ((d.mode == 1 || d.mode == 2) && (!WIDE || uex + units + pp.tail_units > total_units)) {
        d.mode = 4;   // narrow kernels: every 33 <= N <= 128 unit is a 1-patch task; wide: the tail zone
        d.L = 32;
        d.G = 1;
      }
      const uint32_t tasks = (uint32_t)((3ull * d.P + d.G - 1) / d.G);
      if (d.mode != 3) t0 = tasks; else t1 = tasks;
      c.file_off = d.file_off;
      c.out_off = d.out_off;
      c.data_len = d.data_len;
      c.W = d.W;
      c.H = d.H;
      c.gx = d.gx;
      c.P = d.P;
      c.N = (uint8_t)d.N;
      c.mode = (uint8_t)d.mode;
      c.G = (uint8_t)d.G;
      c.L = (uint8_t)d.L;
    }
    a1d[lane] = c;
  }
  uint32_t i0 = t0, i1 = t1;   // inclusive scans over the warp (lanes >= n add 0)
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t v0 = __shfl_up_sync(0xffffffffu, i0, o), v1 = __shfl_up_sync(0xffffffffu, i1, o);
    if (lane >= o) {
      i0 += v0;
      i1 += v1;
    }
  }
  if (lane < pp.n) {
    pre0[lane] = i0 - t0;
    pre1[lane] = i1 - t1;
  }
  if (lane == 31) {
    pre0[pp.n] = i0;
    pre1[pp.n] = i1;
  }
}

template <bool F32, bool WIDE, bool CROP, bool HWC = false>
__global__ void __launch_bounds__(kWarpsPerCta * 32, WIDE ? 4 : (CROP ? L3_CROP_MIN_CTAS : L3_MIN_CTAS))
    l3_decode_kernel(DecodeParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ unsigned int ticket;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* ring = smem + warp * kRingPitch;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kWarpsPerCta * kRingPitch) + warp * kSlots;
  if (lane == 0) {
    for (int s = 0; s < kSlots; s++) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  if (L3_UNPACK_TAB) {
    if (L3_KTAB_RING) {   // this warp's copy, after its ring
      if (lane < 16) {
        const uint32_t k = (uint32_t)lane;
        reinterpret_cast<uint4*>(ring + kKtabOff)[k] =
            (k >= 1 && k <= 8) ? make_uint4(32u - k, 16u - 2u * k, 2u * k, ((1u << k) - 1u) << 16)
                               : make_uint4(0u, 0u, 0u, 0u);
      }
    } else {
      init_ktab();
      __syncthreads();
    }
  }
  __syncwarp();
  uint32_t phase_bits = 0;
  WsHead* head = p.pp.ws.head;

  // shared prefix copy (large batches) or the a1-in-CTA results (small batches): pre0 [34], pre1 [34]
  // u32, then 32 compact descriptors at byte 272 (1808 of the 2056 bytes)
  __shared__ uint64_t sh_prefix[kShPrefix + 1];
  uint32_t* const a1_pre0 = reinterpret_cast<uint32_t*>(sh_prefix);
  uint32_t* const a1_pre1 = a1_pre0 + 34;
  A1Compact* const a1_desc = reinterpret_cast<A1Compact*>(sh_prefix + 34);
  const bool a1in = !CROP && p.a1in != 0;
  if (a1in) {   // a1 inside this CTA (launch_decode_batch: n <= kA1InMaxN, no a1 launch)
    if (warp == 0) a1_in_cta<WIDE>(p.pp, lane, a1_pre0, a1_pre1, a1_desc);
    __syncthreads();
  } else {
    // ---- a1 ran in the preceding l3_prep_kernel (PDL): wait until its results are visible
    pdl_wait();
  }

  const uint64_t* prefix = p.pp.ws.prefix[0];
#if L3_SMEM_PREFIX
  // task -> image lookup from a shared-memory copy of the task prefix (batches of <= 256 images)
  const bool pref_smem = !a1in && p.pp.n <= kShPrefix;
  if (pref_smem) {
    for (int i = threadIdx.x; i <= p.pp.n; i += blockDim.x) sh_prefix[i] = __ldcg(&prefix[i]);
    __syncthreads();
  }
#endif
  const uint64_t total_tasks = a1in ? (uint64_t)a1_pre0[p.pp.n] : prefix[p.pp.n];
  const uint64_t lim = p.pp.src_offsets[p.pp.n] & ~15ull;
  const uint32_t K = p.key_scale;

  // the first task of every warp is its grid-wide warp index (no claim burst on the counter at the
  // start); later tasks come from the dynamic counter, offset by the grid's warp count
  const uint64_t grid_warps = (uint64_t)gridDim.x * kWarpsPerCta;
  uint64_t task = (uint64_t)blockIdx.x * kWarpsPerCta + warp;
  while (task < total_tasks) {
    int lo = 0, hi = p.pp.n;
    if (a1in) {
      while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (a1_pre0[mid] <= task) lo = mid; else hi = mid;
      }
    } else
#if L3_SMEM_PREFIX
    if (pref_smem) {
      while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (sh_prefix[mid] <= task) lo = mid; else hi = mid;
      }
    } else
#endif
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (__ldcg(&prefix[mid]) <= task) lo = mid; else hi = mid;
    }
    const int img = lo;
    const ImgDesc d = a1in ? a1_expand(a1_desc[img]) : p.pp.ws.desc[img];
    const uint32_t t = (uint32_t)(task - (a1in ? (uint64_t)a1_pre0[img] : prefix[img]));
    // claim the next task now; the atomic's latency hides behind this one
    uint64_t next = 0;
    if (lane == 0) next = grid_warps + atomicAdd(&head->next_task[0], 1ull);

    if (WIDE && (d.mode == 1 || d.mode == 2)) {   // u8 out, 33 <= N <= 128: wide 8-column lanes
      phase_bits = (d.mode == 1) ? decode_task8<F32, 4>(p, d, img, t, ring, bars, phase_bits, lim, K)
                                 : decode_task8<F32, 2>(p, d, img, t, ring, bars, phase_bits, lim, K);
      task = __shfl_sync(0xffffffffu, next, 0);
      continue;
    }
    // mode 0 (N <= 32): G >= 4 short patches per warp, each staged whole;
    // mode 4 (33 <= N <= 128 with fp32 out, or the u8 tail zone): one patch per
    // warp, 4 columns per lane, streamed
    const uint32_t G = d.G;
    const bool stream = (G == 1);   // mode 4 (G == 1) vs mode 0 (G >= 4)
    const uint32_t Lw = stream ? 32u : d.L;            // G == 1: the unit spans the warp
    const uint32_t seg = stream ? 0u : lane / Lw, j = stream ? (uint32_t)lane : lane % Lw;
    const uint32_t nunits = 3u * d.P;
    const uint32_t v = t * G + seg;   // unit of the task's image (crop: among the window's units)
    const uint8_t* file = p.pp.src + d.file_off;

    bool active = (seg < G) && (v < (CROP ? 3u * d.gxw * d.gyw : nunits));
    uint32_t w = 0, h = 0, x0 = 0, y0 = 0, ch = 0, u = v;
    uint64_t start = 0, end = 0;
    if (active) {
      uint32_t px, py;
      if (CROP) {   // f3: unit v of the touched sub-grid -> channel, patch
        const uint32_t per = d.gxw * d.gyw;
        ch = v / per;
        const uint32_t rem = v - ch * per;
        py = d.py0 + rem / d.gxw;
        px = d.px0 + rem % d.gxw;
        u = ch * d.P + py * d.gx + px;
      } else {
        ch = u / d.P;
        const uint32_t pp = u - ch * d.P;
        px = pp % d.gx;
        py = pp / d.gx;
      }
      x0 = px * d.N;
      y0 = py * d.N;
      w = min(d.N, d.W - x0);
      h = min(d.N, d.H - y0);
      if (CROP) {   // f3: skip patches outside the window; rows below it are not needed
        if (x0 + w <= d.cx || x0 >= d.cx + d.cw || y0 + h <= d.cy || y0 >= d.cy + d.ch) active = false;
        else h = min(h, d.cy + d.ch - y0);
      }
    }
    if (active) {
      const uint64_t off = ld_u32le(file + 13 + 4ull * u);
      const uint64_t nxt = (u + 1 < nunits) ? (uint64_t)ld_u32le(file + 17 + 4ull * u) : d.data_len;
      if (unit_offsets_bad(u, nunits, off, nxt, d.data_len)) {
        if (j == 0) record_err(&p.pp.ws.errkey[img], 0u);   // header-level: CORRUPT_HEADER
        active = false;
      } else {
        start = d.data_off + off;
        end = d.data_off + nxt;
      }
    }
    const uint32_t worst = active ? worst_patch_bytes(w, h) : 0u;
    const uint64_t stage_end = active ? min(end, start + worst + 8) : 0;

    LaneRows s;
    s.w = w;
    s.h = active ? h : 0u;
    s.j4 = 4u * j;
    s.first = (j == 0);
    s.last = (s.j4 + 4u >= w);
    s.valid = active && (s.j4 < w);
    s.kacc = 0;
    s.A = s.B = 0;
    s.Q = 0;
    if (!F32 && L3_PRED4 != 0 && L3_H2_U8 == 0) {   // byte-form predictor: (left Q, Q) and (Q, right Q) selectors
      s.selL = s.first ? 0x6544u : 0x6543u;
      s.selR = s.last ? 0x3321u : 0x4321u;
    } else {                         // L3_EDGE_SEL: TLA = prmt(left B, A, selL), TRB = prmt(B, right A, selR)
      s.selL = s.first ? 0x5454u : 0x5452u;
      s.selR = s.last ? 0x5212u : 0x5412u;
    }
    s.selG = (w >= s.j4 + 4u) ? 0x3210u : (w == s.j4 + 3u) ? 0x2210u : (w == s.j4 + 2u) ? 0x1110u : 0x0000u;
    const uint32_t esz = F32 ? 4u : 1u;
    if (CROP) {   // augment variant (f3): window, flip; planar, or HWC (interleaved channels)
      const bool flip = HWC ? (d.flip & 1u) != 0 : d.flip != 0;
      const int32_t cw = (int32_t)d.cw, cj0 = (int32_t)(x0 + s.j4) - (int32_t)d.cx;
      const int32_t bc = flip ? cw - 4 - cj0 : cj0;   // window column of the lane's lowest-address element
      const int64_t stride = (HWC ? 3 : 1) * (int64_t)esz;
      s.ri = (int32_t)y0 - (int32_t)d.cy;
      s.chh = d.ch;
      s.pitch = (uint32_t)(cw * stride);
      s.optr = reinterpret_cast<uint8_t*>(p.out) +
               (int64_t)(d.out_off + (HWC ? (uint64_t)ch : (uint64_t)ch * d.ch * d.cw)) * esz +
               ((int64_t)s.ri * cw + bc) * stride;
      s.qsel = flip ? 0x0123u : 0x3210u;
      s.cmask = 0;
#pragma unroll
      for (int t = 0; t < 4; t++) {
        const int32_t c = flip ? 3 - t : t;   // lane column of output slot t
        if (active && s.j4 + (uint32_t)c < w && cj0 + c >= 0 && cj0 + c < cw) s.cmask |= 1u << t;
      }
    } else {
      const uint64_t elem = d.out_off + (uint64_t)ch * d.W * d.H + (uint64_t)y0 * d.W + x0 + s.j4;
      s.optr = reinterpret_cast<uint8_t*>(p.out) + elem * esz;
      s.pitch = d.W * esz;
    }
    const uint32_t len = active ? (uint32_t)min((uint64_t)(worst + 16), end - start) : 0u;

    StreamState st;
    st.landed_end = 0xFFFFFFFFu;
    if (!stream) {
      // whole-task staging: one aligned window per segment, one barrier (bars[0])
      const uint32_t seg_bytes = kRingBytes / G;
      uint32_t bytes = 0;
      uint64_t a16 = 0, b16 = 0;
      s.bp = 0;
      if (active) {
        a16 = start & ~15ull;
        b16 = (stage_end + 15) & ~15ull;
        const uint64_t be = b16 < lim ? b16 : lim;
        bytes = be > a16 ? (uint32_t)(be - a16) : 0u;
        s.bp = seg * seg_bytes * 8u + (uint32_t)(start - a16) * 8u;
      }
      uint32_t tx = (active && j == 0) ? bytes : 0u;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) tx += __shfl_xor_sync(0xffffffffu, tx, o);
      if (lane == 0) mbar_arrive_expect_tx(&bars[0], tx);
      __syncwarp();
      if (active) {
        uint8_t* dst = ring + seg * seg_bytes;
        if (j == 0 && bytes) bulk_g2s(dst, p.pp.src + a16, bytes, &bars[0]);
        const uint64_t t0 = a16 > lim ? a16 : lim;
        for (uint64_t x = t0 + j; x < stage_end && x < b16; x += Lw) dst[x - a16] = __ldg(p.pp.src + x);
      }
      mbar_wait(&bars[0], phase_bits & 1u);
      phase_bits ^= 1u;
      __syncwarp();
      if (active) swap_words(ring + seg * seg_bytes, 0, (uint32_t)(b16 - a16), j, Lw);
      __syncwarp();
    } else {
      // stream the unit through the ring: chunk i of [A, B) -> slot i % kSlots
      st.A = start & ~15ull;
      st.B = (stage_end + 15) & ~15ull;
      st.stage_end = stage_end;
      if (F32) stream_rel_init(st, lim);
      constexpr int SB = kStreamSB<F32>(), SS = kStreamSlots<F32>();
      st.nchunks = active ? (uint32_t)((st.B - st.A + SB - 1) / SB) : 0u;
      st.issued = 0;
      st.landed = 0;
      st.landed_end = 0;
      const uint32_t first = min(st.nchunks, (uint32_t)SS);
#if L3_BULK_FIRST
      // the first `first` chunks are contiguous in the ring: one bulk copy on bars[0]
      if (first > 0) {   // (no arrive on bars[0] without a matching wait)
        stage_range(p.pp.src, st.A, min(st.A + (uint64_t)first * SB, st.B), lim, st.stage_end, ring,
                    &bars[0], lane == 0, lane, 32);
        st.issued = first;
        st.group = first;
      }
#else
      while (st.issued < first) stream_issue<SS, F32 && L3_ISSUE_REL != 0, SB>(p.pp.src, lim, st, ring, bars, lane);
#endif
      __syncwarp();
      s.bp = (uint32_t)(start - st.A) * 8u;
    }
    s.lim = s.bp + len * 8u;

    uint32_t hmax = s.h;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) hmax = max(hmax, __shfl_xor_sync(0xffffffffu, hmax, o));
    const bool fast_ok = !active || ((w & 3u) == 0 && (CROP || (((reinterpret_cast<uintptr_t>(s.optr) &
                                                                   (F32 ? 15 : 3)) == 0) &&
                                                                 ((s.pitch & (F32 ? 15u : 3u)) == 0))));
    const bool fast = __all_sync(0xffffffffu, fast_ok);
    // u8: whole 16-byte lane groups (patch width a multiple of 16, 16-byte aligned rows) store 128 bits
    s.v16 = !F32 && !CROP && L3_U8_V16 != 0 &&
            __all_sync(0xffffffffu, !active || ((w & 15u) == 0 && ((reinterpret_cast<uintptr_t>(s.optr) - s.j4) & 15u) == 0 &&
                                                (s.pitch & 15u) == 0));
    // u8 narrow variant, whole-staged N <= 32 tasks (small mixed-shape images, e.g. C2): planar
    // output that is not vector-aligned (image width not a multiple of 4) but has no ragged patch
    // takes scalar stores without per-column tests or edge ghosts. Everything else keeps two paths
    // (code size, registers: a third instantiation on the streamed path cost C3 5 %).
    constexpr bool kAlignedOnlyPath = !F32 && !WIDE && !CROP;
    const bool aligned_only = kAlignedOnlyPath && !fast && __all_sync(0xffffffffu, !active || (w & 3u) == 0);
    const float sc = F32 ? (ch == 0 ? p.scale[0] : (ch == 1 ? p.scale[1] : p.scale[2])) : 0.f;
    const float bi = F32 ? (ch == 0 ? p.bias[0] : (ch == 1 ? p.bias[1] : p.bias[2])) : 0.f;
    const uint32_t rowmax = (12u + 8u * 128u) / 8u + 10u;
    if (hmax > 0) {
      if (stream) {
        if (fast)
          decode_unit_rows<F32, true, true, CROP, HWC>(s, ring, hmax, Lw, sc, bi, K, p.pp.src, lim, st, bars, phase_bits, rowmax, lane);
        else
          decode_unit_rows<F32, false, true, CROP, HWC>(s, ring, hmax, Lw, sc, bi, K, p.pp.src, lim, st, bars, phase_bits, rowmax, lane);
      } else {
        if (fast)
          decode_unit_rows<F32, true, false, CROP, HWC>(s, ring, hmax, Lw, sc, bi, K, p.pp.src, lim, st, bars, phase_bits, rowmax, lane);
        else if constexpr (kAlignedOnlyPath) {
          if (aligned_only)
            decode_unit_rows<F32, false, false, CROP, HWC, false>(s, ring, hmax, Lw, sc, bi, K, p.pp.src, lim, st, bars, phase_bits, rowmax, lane);
          else
            decode_unit_rows<F32, false, false, CROP, HWC>(s, ring, hmax, Lw, sc, bi, K, p.pp.src, lim, st, bars, phase_bits, rowmax, lane);
        }
        else
          decode_unit_rows<F32, false, false, CROP, HWC>(s, ring, hmax, Lw, sc, bi, K, p.pp.src, lim, st, bars, phase_bits, rowmax, lane);
      }
    }
    const bool err = active && (s.kacc >= 0x80000000u || s.bp > s.lim);
    if (__any_sync(0xffffffffu, err) && err && j == 0) {   // a7: exact first error of a failed unit
      const int code = unit_first_error(p.pp.src, start, end, w, h);
      if (code != L3_OK) record_err(&p.pp.ws.errkey[img], err_key(u, code));
    }
    if (stream) {   // drain copies that were issued but never waited for
      while (st.landed < st.issued) {
        stream_land<kStreamSlots<F32>()>(st, bars, phase_bits);
        st.landed++;
      }
    }
    __syncwarp();
    fence_proxy_async_smem();
    task = __shfl_sync(0xffffffffu, next, 0);
  }

  // ---- N > 128 units (never chosen by the policy): generic path, same ring
  const uint64_t total1 = a1in ? (uint64_t)a1_pre1[p.pp.n] : p.pp.ws.prefix[1][p.pp.n];
  if (total1 > 0) {
    GenericArgs ga;
    ga.src = p.pp.src;
    ga.prefix1 = p.pp.ws.prefix[1];
    ga.desc = p.pp.ws.desc;
    ga.a1_pre1 = a1in ? a1_pre1 : nullptr;
    ga.a1_desc = a1in ? a1_desc : nullptr;
    ga.errkey = p.pp.ws.errkey;
    ga.out = p.out;
    ga.lim = lim;
    ga.n = p.pp.n;
    for (int c = 0; c < 3; c++) {
      ga.scale[c] = p.scale[c];
      ga.bias[c] = p.bias[c];
    }
    for (;;) {
      uint64_t t1 = 0;
      if (lane == 0) t1 = atomicAdd(&head->next_task[1], 1ull);
      t1 = __shfl_sync(0xffffffffu, t1, 0);
      if (t1 >= total1) break;
      phase_bits = generic_task<F32, CROP, HWC>(ga, t1, ring, bars, phase_bits);
    }
  }

  // ---- a7: per-image status, by the last CTA
  a7_finish(p.pp, head, &ticket, a1in ? a1_desc : nullptr);
}

}  // namespace l3
