// l3_decode_wide8.cuh — "wide lane" decode path for 33 <= N <= 128 (included by
// l3_decode_fast.cuh). Each lane owns 8 consecutive columns (4 pairs), so a
// patch row of up to 128 columns needs 16 lanes and a warp decodes G = 2
// patches at once (G = 4 for N <= 64). Per-row overhead that does not scale
// with the column count (header fetch, ring test, shuffles, loop, store
// address) is paid once per 8 columns instead of once per 4 — the kernel is
// issue-bound, so this is the lever.
//
// Each segment (one patch) streams its own compressed range through its own
// ring of SLOTS x 1 KB TMA bulk-copy slots (+16-byte wrap mirror); the two or
// four streams of a warp progress independently, so ring bookkeeping runs per
// segment under the segment's lane mask.
#pragma once

namespace l3 {

constexpr int kW8Pitch = kRingBytes + 64;   // per-warp ring region: up to 4 segment rings + mirrors

// Byte offset of segment `seg`'s ring inside the warp's region.
template <int SLOTS>
__device__ __forceinline__ uint32_t w8_ring_off(uint32_t seg) {
  return seg * (SLOTS * kSlotBytes + 16);
}

// 64 stream bits at unwrapped bit position `bit` of a pre-swapped ring of
// SLOTS KB (+ mirror): hi = bits [bit, bit+32), lo = bits [bit+32, bit+64).
template <int SLOTS>
__device__ __forceinline__ void w8_bits64(const uint8_t* ring, uint32_t bit, uint32_t& hi, uint32_t& lo) {
  const uint32_t* p = reinterpret_cast<const uint32_t*>(ring + ((bit >> 3) & (uint32_t)(SLOTS * kSlotBytes - 4)));
  const uint32_t w0 = p[0], w1 = p[1], w2 = p[2];   // p[1], p[2] may be the mirror
  asm("shf.l.wrap.b32 %0, %1, %2, %3;" : "=r"(hi) : "r"(w1), "r"(w0), "r"(bit));
  asm("shf.l.wrap.b32 %0, %1, %2, %3;" : "=r"(lo) : "r"(w2), "r"(w1), "r"(bit));
}

template <int SLOTS>
__device__ __forceinline__ uint32_t w8_bits32(const uint8_t* ring, uint32_t bit) {
  const uint32_t* p = reinterpret_cast<const uint32_t*>(ring + ((bit >> 3) & (uint32_t)(SLOTS * kSlotBytes - 4)));
  uint32_t d;
  asm("shf.l.wrap.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(p[1]), "r"(p[0]), "r"(bit));
  return d;
}

__device__ __forceinline__ uint32_t shf_l_clamp(uint32_t lo, uint32_t hi, uint32_t n) {
  uint32_t d;
  asm("shf.l.clamp.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(lo), "r"(hi), "r"(n));
  return d;
}

// Stream state of one segment (uniform over the segment's lanes).
struct Seg8 {
  uint64_t A, B, stage_end;
  uint32_t nchunks, issued, landed, landed_end;
  uint32_t relB, rel_bulk, rel_end;   // A-relative bounds (stream_rel_init)
};

template <int SLOTS>
__device__ __forceinline__ void w8_issue(const uint8_t* src, uint64_t lim, Seg8& s, uint8_t* ring, uint64_t* bars,
                                         uint32_t j, uint32_t L) {
#if L3_ISSUE_REL
  stream_issue_rel<SLOTS>(src, s, ring, bars, j == 0, j, L);
#else
  const uint32_t c = s.issued;
  const uint64_t ca = s.A + (uint64_t)c * kSlotBytes;
  const uint64_t cb = min(ca + kSlotBytes, s.B);
  stage_range(src, ca, cb, lim, s.stage_end, ring + (c % SLOTS) * kSlotBytes, &bars[c % SLOTS], j == 0, (int)j,
              (int)L);
  s.issued = c + 1;
#endif
}

// Refill consumed slots, then wait (and byte-swap) until `need` A-relative bytes
// are resident. Collective over the segment's lanes (`mask`).
template <int SLOTS>
__device__ __forceinline__ void w8_advance(const uint8_t* src, uint64_t lim, Seg8& s, uint8_t* ring, uint64_t* bars,
                                           uint32_t& phase, uint32_t consumed_byte, uint32_t need, uint32_t j,
                                           uint32_t L, uint32_t mask) {
  const uint32_t consumed = consumed_byte / kSlotBytes;
  if (s.issued < s.nchunks && s.issued < consumed + SLOTS) {
    __syncwarp(mask);
    fence_proxy_async_smem();
    while (s.issued < s.nchunks && s.issued < consumed + SLOTS) w8_issue<SLOTS>(src, lim, s, ring, bars, j, L);
    __syncwarp(mask);
  }
  while (s.landed < s.issued && (uint64_t)s.landed * kSlotBytes < need) {
    const uint32_t sl = s.landed % SLOTS;
    mbar_wait(&bars[sl], (phase >> sl) & 1u);
    phase ^= 1u << sl;
    __syncwarp(mask);
    swap_words(ring, sl * kSlotBytes, (sl + 1) * kSlotBytes, j, L);
    __syncwarp(mask);
    if (sl == 0) {
      if (j < 4) reinterpret_cast<uint32_t*>(ring + SLOTS * kSlotBytes)[j] = reinterpret_cast<uint32_t*>(ring)[j];
      __syncwarp(mask);
    }
    s.landed++;
  }
  s.landed_end = (s.landed == s.nchunks) ? 0xFFFFFFFFu : s.landed * kSlotBytes;
}

// Row state of one lane: 8 consecutive columns j8..j8+7 as 4 pairs.
struct Lane8 {
  uint32_t bp, lim, w, h, j8, raw, kacc;
  bool first, last, valid;
  bool v16;   // u8 FAST: 128-bit stores (lane 2m gathers lane 2m+1's 8 bytes), rows 16-byte aligned
  uint8_t* optr;
  uint32_t pitch;
  uint32_t A, B, C, D;
};

// Unpack 4 deltas (top-aligned k-bit fields of `f`) into two pairs, + base.
__device__ __forceinline__ void unpack4(uint32_t f, uint32_t sh, uint32_t pk, uint32_t pk2, uint32_t pk3,
                                        uint32_t base2, uint32_t& dA, uint32_t& dB) {
  const uint32_t d0 = shr_c(f, sh);
  const uint32_t d1 = shr_c(f * pk, sh);
  const uint32_t d2 = shr_c(f * pk2, sh);
  const uint32_t d3 = shr_c(f * pk3, sh);
  dA = d1 * 0x10000u + d0 + base2;
  dB = d3 * 0x10000u + d2 + base2;
}

template <bool F32, bool FAST>
__device__ __forceinline__ void store8(const Lane8& s, uint32_t xA, uint32_t xB, uint32_t xC, uint32_t xD, float sc,
                                       float bi, bool pred, uint32_t L) {
  if (F32) {
    const float v0 = fmaf((float)(xA & 0xFFFFu), sc, bi), v1 = fmaf((float)(xA >> 16), sc, bi);
    const float v2 = fmaf((float)(xB & 0xFFFFu), sc, bi), v3 = fmaf((float)(xB >> 16), sc, bi);
    const float v4 = fmaf((float)(xC & 0xFFFFu), sc, bi), v5 = fmaf((float)(xC >> 16), sc, bi);
    const float v6 = fmaf((float)(xD & 0xFFFFu), sc, bi), v7 = fmaf((float)(xD >> 16), sc, bi);
    if (FAST) {
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %9, 0;\n\t"
          "@p st.global.v4.f32 [%0], {%1, %2, %3, %4};\n\t"
          "@p st.global.v4.f32 [%0+16], {%5, %6, %7, %8};\n\t}" ::"l"(s.optr),
          "f"(v0), "f"(v1), "f"(v2), "f"(v3), "f"(v4), "f"(v5), "f"(v6), "f"(v7), "r"((uint32_t)pred));
    } else if (pred) {
      float* o = reinterpret_cast<float*>(s.optr);
      const float v[8] = {v0, v1, v2, v3, v4, v5, v6, v7};
#pragma unroll
      for (int c = 0; c < 8; c++)
        if (s.j8 + c < s.w) o[c] = v[c];
    }
  } else {
    const uint32_t q0 = prmt(xA, xB, 0x6420), q1 = prmt(xC, xD, 0x6420);
    if (FAST && s.v16) {   // warp-uniform: 128-bit stores by the even lanes
      const uint32_t r0 = __shfl_down_sync(0xffffffffu, q0, 1, L), r1 = __shfl_down_sync(0xffffffffu, q1, 1, L);
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %5, 0;\n\t"
          "@p st.global.v4.b32 [%0], {%1, %2, %3, %4};\n\t}" ::"l"(s.optr), "r"(q0), "r"(q1), "r"(r0), "r"(r1),
          "r"((uint32_t)(pred && (s.j8 & 15u) == 0)));
    } else if (FAST) {
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %3, 0;\n\t"
          "@p st.global.v2.b32 [%0], {%1, %2};\n\t}" ::"l"(s.optr), "r"(q0), "r"(q1), "r"((uint32_t)pred));
    } else if (pred) {
      uint8_t* o = s.optr;
#pragma unroll
      for (int c = 0; c < 8; c++)
        if (s.j8 + c < s.w) o[c] = (uint8_t)((c < 4 ? q0 : q1) >> (8 * (c & 3)));
    }
  }
}

#ifndef L3_PRED4_WIDE
#define L3_PRED4_WIDE 0   // 1: byte-form predictor on the u8 wide path (A/B option)
#endif

// u8 store of the lane's 8 samples in byte form.
template <bool FAST>
__device__ __forceinline__ void store8q(const Lane8& s, uint32_t q0, uint32_t q1, bool pred) {
  if (FAST) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %3, 0;\n\t"
        "@p st.global.v2.b32 [%0], {%1, %2};\n\t}" ::"l"(s.optr), "r"(q0), "r"(q1), "r"((uint32_t)pred));
  } else if (pred) {
    uint8_t* o = s.optr;
#pragma unroll
    for (int c = 0; c < 8; c++)
      if (s.j8 + c < s.w) o[c] = (uint8_t)((c < 4 ? q0 : q1) >> (8 * (c & 3)));
  }
}

// One row of one lane (a3-a6) — see decode_row in l3_decode_fast.cuh for the
// validity accumulation; this is the same step on 8 columns.
template <bool FIRST, bool F32, bool FAST, bool GUARD, int SLOTS>
__device__ __forceinline__ void decode_row8(Lane8& s, const uint8_t* ring, uint32_t r, uint32_t L, float sc,
                                            float bi, uint32_t K) {
  const uint32_t k = s.raw >> 28;
  const uint32_t base2 = (s.raw >> 20) * 0x00010001u;
  const uint32_t rowbits = 12u + k * s.w;
  const bool live = GUARD ? (r < s.h) : true;
  const uint32_t nbp = s.bp + rowbits;
  const uint32_t raw_next = w8_bits32<SLOTS>(ring, nbp);   // next row's header, fetched early
  // a4: 8 k-bit deltas of this lane, 8k <= 64 bits
  uint32_t f0, f1;
  w8_bits64<SLOTS>(ring, s.bp + 12u + s.j8 * k, f0, f1);
  const uint32_t g1 = shf_l_clamp(f1, f0, 4u * k);        // deltas 4..7 top-aligned
  const uint32_t sh = 32u - k;
  const uint32_t pk = shl_c(1u, k), pk2 = pk * pk, pk3 = pk2 * pk;
  uint32_t dA, dB, dC, dD;
  unpack4(f0, sh, pk, pk2, pk3, base2, dA, dB);
  unpack4(g1, sh, pk, pk2, pk3, base2, dC, dD);
  uint32_t xA, xB, xC, xD;
  if constexpr (!F32 && L3_PRED4_WIDE != 0) {
    // byte-form predictor (paeth_pred4), state s.A = [c0..c3], s.B = [c4..c7]
    if (FIRST) {
      xA = dA;
      xB = dB;
      xC = dC;
      xD = dD;
    } else {
      const uint32_t Lq = __shfl_up_sync(0xffffffffu, s.B, 1, L);     // left lane's [c-4 .. c-1]
      const uint32_t Rq = __shfl_down_sync(0xffffffffu, s.A, 1, L);   // right lane's [c8 .. c11]
      const uint32_t L0 = prmt(Lq, s.A, 0x6543u + (uint32_t)s.first);           // [c-1 c0 c1 c2] (C4)
      const uint32_t R0 = prmt(s.A, s.B, 0x4321u);                               // [c1 c2 c3 c4]
      const uint32_t L1 = prmt(s.A, s.B, 0x6543u);                               // [c3 c4 c5 c6]
      const uint32_t R1 = prmt(s.B, Rq, 0x4321u - ((uint32_t)s.last << 12));     // [c5 c6 c7 c8] (C4)
      const uint32_t p0 = paeth_pred4(L0, s.A, R0), p1 = paeth_pred4(L1, s.B, R1);
      xA = prmt(p0, 0u, 0x4140u) + dA;
      xB = prmt(p0, 0u, 0x4342u) + dB;
      xC = prmt(p1, 0u, 0x4140u) + dC;
      xD = prmt(p1, 0u, 0x4342u) + dD;
    }
    uint32_t q0 = prmt(xA, xB, 0x6420u), q1 = prmt(xC, xD, 0x6420u);
    if (!FAST) {   // ragged patch: columns >= w are ghosts of column w-1
      uint32_t x[8];
#pragma unroll
      for (int c = 0; c < 8; c++) x[c] = ((c < 4 ? q0 : q1) >> (8 * (c & 3))) & 0xFFu;
#pragma unroll
      for (int c = 1; c < 8; c++)
        if (s.j8 + c >= s.w) x[c] = x[c - 1];
      q0 = x[0] | (x[1] << 8) | (x[2] << 16) | (x[3] << 24);
      q1 = x[4] | (x[5] << 8) | (x[6] << 16) | (x[7] << 24);
    }
    store8q<FAST>(s, q0, q1, live && s.valid);
    s.A = q0;
    s.B = q1;
    if (live) {
      s.kacc = max(s.kacc, s.raw - 0x10000000u);
      s.bp = nbp;
      s.raw = raw_next;
    }
    s.optr += s.pitch;
    return;
  }
  // which of the 4 pairs run the biased-half predictor (paeth_h2, FMA pipes; bit i = pair i); any
  // non-zero mask keeps every sample as a biased half 0x6400 | c (l3_decode_fast.cuh)
  constexpr int kH2 = F32 ? 0 : L3_H2_WIDE;
  constexpr uint32_t kBias = kH2 ? 0x64006400u : 0u;
  if (FIRST) {
    xA = kH2 ? lo_bytes_biased(dA, bias_reg(K)) : (dA & 0x00FF00FFu);
    xB = kH2 ? lo_bytes_biased(dB, bias_reg(K)) : (dB & 0x00FF00FFu);
    xC = kH2 ? lo_bytes_biased(dC, bias_reg(K)) : (dC & 0x00FF00FFu);
    xD = kH2 ? lo_bytes_biased(dD, bias_reg(K)) : (dD & 0x00FF00FFu);
  } else {
    // a5: row-wise parallel custom Paeth, 4 pairs
    const uint32_t Dl = __shfl_up_sync(0xffffffffu, s.D, 1, L);     // left lane's (c6, c7)
    const uint32_t Ar = __shfl_down_sync(0xffffffffu, s.A, 1, L);   // right lane's (c0, c1)
    const uint32_t LF = s.first ? (s.A << 16) : Dl;   // byte 2 = TL of column j8 (reading C4)
    const uint32_t RT = s.last ? (s.D >> 16) : Ar;    // byte 0 = TR of column j8+7 (reading C4)
    const uint32_t TLA = prmt(LF, s.A, 0x5452);
    const uint32_t TRA = prmt(s.A, s.B, 0x5412);
    const uint32_t TRB = prmt(s.B, s.C, 0x5412);
    const uint32_t TRC = prmt(s.C, s.D, 0x5412);
    const uint32_t TRD = prmt(s.D, RT, 0x5412);
    const uint32_t pA = (kH2 & 1) ? paeth_h2(TLA, s.A, TRA) : paeth_pred2(TLA, s.A, TRA, K);
    const uint32_t pB = (kH2 & 2) ? paeth_h2(TRA, s.B, TRB) : paeth_pred2(TRA, s.B, TRB, K);
    const uint32_t pC = (kH2 & 4) ? paeth_h2(TRB, s.C, TRC) : paeth_pred2(TRB, s.C, TRC, K);
    const uint32_t pD = (kH2 & 8) ? paeth_h2(TRC, s.D, TRD) : paeth_pred2(TRC, s.D, TRD, K);
    xA = kH2 ? lo_bytes_biased(pA + dA, bias_reg(K)) : ((pA + dA) & 0x00FF00FFu);
    xB = kH2 ? lo_bytes_biased(pB + dB, bias_reg(K)) : ((pB + dB) & 0x00FF00FFu);
    xC = kH2 ? lo_bytes_biased(pC + dC, bias_reg(K)) : ((pC + dC) & 0x00FF00FFu);
    xD = kH2 ? lo_bytes_biased(pD + dD, bias_reg(K)) : ((pD + dD) & 0x00FF00FFu);
  }
  if (!FAST) {   // ragged patch: columns >= w are ghosts of column w-1
    uint32_t x[8] = {xA & 0xFFu, (xA >> 16) & 0xFFu, xB & 0xFFu, (xB >> 16) & 0xFFu,
                     xC & 0xFFu, (xC >> 16) & 0xFFu, xD & 0xFFu, (xD >> 16) & 0xFFu};
#pragma unroll
    for (int c = 1; c < 8; c++)
      if (s.j8 + c >= s.w) x[c] = x[c - 1];
    xA = x[0] | (x[1] << 16) | kBias;
    xB = x[2] | (x[3] << 16) | kBias;
    xC = x[4] | (x[5] << 16) | kBias;
    xD = x[6] | (x[7] << 16) | kBias;
  }
  store8<F32, FAST>(s, xA, xB, xC, xD, sc, bi, live && s.valid, L);
  s.A = xA;
  s.B = xB;
  s.C = xC;
  s.D = xD;
  if (live) {
    s.kacc = max(s.kacc, s.raw - 0x10000000u);
    s.bp = nbp;
    s.raw = raw_next;
  }
  s.optr += s.pitch;
}

template <bool F32, bool FAST, bool GUARD, int SLOTS>
__device__ __forceinline__ void decode_rows8(Lane8& s, uint8_t* ring, uint32_t hmax, uint32_t L, float sc, float bi,
                                             uint32_t K, const uint8_t* src, uint64_t lim, Seg8& st,
                                             uint64_t* bars, uint32_t& phase, uint32_t j, uint32_t mask) {
  const uint32_t rowmax = (12u + 8u * 128u) / 8u + 12u;
  // the ring test is per segment (segments progress independently); lanes of a
  // finished segment (r >= h) stop testing
  if ((s.bp >> 3) + 2u * rowmax > st.landed_end && s.h > 0)
    w8_advance<SLOTS>(src, lim, st, ring, bars, phase, s.bp >> 3, (s.bp >> 3) + 2u * rowmax, j, L, mask);
  s.raw = w8_bits32<SLOTS>(ring, s.bp);
  decode_row8<true, F32, FAST, GUARD, SLOTS>(s, ring, 0, L, sc, bi, K);
  uint32_t r = 1;
  for (; r + 1 < hmax; r += 2) {
    if ((s.bp >> 3) + 2u * rowmax > st.landed_end && r < s.h)
      w8_advance<SLOTS>(src, lim, st, ring, bars, phase, s.bp >> 3, (s.bp >> 3) + 2u * rowmax, j, L, mask);
    decode_row8<false, F32, FAST, GUARD, SLOTS>(s, ring, r, L, sc, bi, K);
    decode_row8<false, F32, FAST, GUARD, SLOTS>(s, ring, r + 1, L, sc, bi, K);
  }
  if (r < hmax) {
    if ((s.bp >> 3) + rowmax > st.landed_end && r < s.h)
      w8_advance<SLOTS>(src, lim, st, ring, bars, phase, s.bp >> 3, (s.bp >> 3) + rowmax, j, L, mask);
    decode_row8<false, F32, FAST, GUARD, SLOTS>(s, ring, r, L, sc, bi, K);
  }
}

// One wide-lane task: G = 32 / L units (u0 .. u0+G-1) of image `img`.
// Returns the warp's updated per-barrier phase bits.
template <bool F32, int SLOTS>
__device__ __forceinline__ uint32_t decode_task8(const DecodeParams& p, const ImgDesc& d, int img, uint32_t t,
                                                 uint8_t* wring, uint64_t* wbars, uint32_t phase_bits, uint64_t lim,
                                                 uint32_t K) {
  constexpr uint32_t G = 8 / SLOTS;          // SLOTS = 4 -> 2 segments of 16 lanes; SLOTS = 2 -> 4 of 8
  constexpr uint32_t L = 32 / G;
  const int lane = threadIdx.x & 31;
  const uint32_t seg = lane / L, j = lane % L;
  const uint32_t mask = ((L == 32) ? 0xffffffffu : ((1u << L) - 1u)) << (seg * L);
  uint8_t* ring = wring + w8_ring_off<SLOTS>(seg);
  uint64_t* bars = wbars + seg * SLOTS;
  uint32_t phase = (phase_bits >> (seg * SLOTS)) & ((1u << SLOTS) - 1u);

  const uint32_t nunits = 3u * d.P;
  const uint32_t u = t * G + seg;
  const uint8_t* file = p.pp.src + d.file_off;
  bool active = u < nunits;
  uint32_t w = 0, h = 0, x0 = 0, y0 = 0, ch = 0;
  uint64_t start = 0, end = 0;
  if (active) {
    ch = u / d.P;
    const uint32_t pp = u - ch * d.P;
    x0 = (pp % d.gx) * d.N;
    y0 = (pp / d.gx) * d.N;
    w = min(d.N, d.W - x0);
    h = min(d.N, d.H - y0);
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
  const uint32_t len = active ? (uint32_t)min((uint64_t)(worst + 16), end - start) : 0u;

  Seg8 st;
  st.A = start & ~15ull;
  st.B = (stage_end + 15) & ~15ull;
  st.stage_end = stage_end;
  stream_rel_init(st, lim);
  st.nchunks = active ? (uint32_t)((st.B - st.A + kSlotBytes - 1) / kSlotBytes) : 0u;
  st.issued = 0;
  st.landed = 0;
  st.landed_end = 0;
  const uint32_t first = min(st.nchunks, (uint32_t)SLOTS);
  while (st.issued < first) w8_issue<SLOTS>(p.pp.src, lim, st, ring, bars, j, L);
  __syncwarp();

  Lane8 s;
  s.bp = (uint32_t)(start - st.A) * 8u;
  s.lim = s.bp + len * 8u;
  s.w = w;
  s.h = active ? h : 0u;
  s.j8 = 8u * j;
  s.first = (j == 0);
  s.last = (s.j8 + 8u >= w);
  s.valid = active && (s.j8 < w);
  s.kacc = 0;
  s.A = s.B = s.C = s.D = 0;
  const uint32_t esz = F32 ? 4u : 1u;
  const uint64_t elem = d.out_off + (uint64_t)ch * d.W * d.H + (uint64_t)y0 * d.W + x0 + s.j8;
  s.optr = reinterpret_cast<uint8_t*>(p.out) + elem * esz;
  s.pitch = d.W * esz;

  uint32_t hmax = s.h, hmin = active ? h : 0xFFFFFFFFu;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    hmax = max(hmax, __shfl_xor_sync(0xffffffffu, hmax, o));
    hmin = min(hmin, __shfl_xor_sync(0xffffffffu, hmin, o));
  }
  const uint32_t align = F32 ? 15u : 7u;
  const bool fast_ok = !active || ((w & 7u) == 0 && ((reinterpret_cast<uintptr_t>(s.optr) & align) == 0) &&
                                   ((s.pitch & align) == 0));
  const bool fast = __all_sync(0xffffffffu, fast_ok);
  s.v16 = !F32 && L3_U8_V16 != 0 &&
          __all_sync(0xffffffffu, !active || ((w & 15u) == 0 && ((reinterpret_cast<uintptr_t>(s.optr) - s.j8) & 15u) == 0 &&
                                              (s.pitch & 15u) == 0));
  const bool guard = hmin != hmax;    // segments of unequal height (or an idle segment)
  const float sc = F32 ? (ch == 0 ? p.scale[0] : (ch == 1 ? p.scale[1] : p.scale[2])) : 0.f;
  const float bi = F32 ? (ch == 0 ? p.bias[0] : (ch == 1 ? p.bias[1] : p.bias[2])) : 0.f;
  if (hmax > 0) {
    if (fast && !guard)
      decode_rows8<F32, true, false, SLOTS>(s, ring, hmax, L, sc, bi, K, p.pp.src, lim, st, bars, phase, j, mask);
    else if (fast)
      decode_rows8<F32, true, true, SLOTS>(s, ring, hmax, L, sc, bi, K, p.pp.src, lim, st, bars, phase, j, mask);
    else
      decode_rows8<F32, false, true, SLOTS>(s, ring, hmax, L, sc, bi, K, p.pp.src, lim, st, bars, phase, j, mask);
  }
  const bool err = active && (s.kacc >= 0x80000000u || s.bp > s.lim);
  if (__any_sync(0xffffffffu, err) && err && j == 0) {   // a7: exact first error of a failed unit
    const int code = unit_first_error(p.pp.src, start, end, w, h);
    if (code != L3_OK) record_err(&p.pp.ws.errkey[img], err_key(u, code));
  }
  // drain copies that were issued but never waited for
  while (st.landed < st.issued) {
    const uint32_t sl = st.landed % SLOTS;
    mbar_wait(&bars[sl], (phase >> sl) & 1u);
    phase ^= 1u << sl;
    st.landed++;
  }
  __syncwarp();
  fence_proxy_async_smem();
  // merge every segment's barrier phases back into the warp-wide phase bits
  const uint32_t mine = phase << (seg * SLOTS);
  const uint32_t segbits = ((1u << SLOTS) - 1u) << (seg * SLOTS);
  const uint32_t merged = __reduce_or_sync(0xffffffffu, (j == 0) ? mine : 0u);
  const uint32_t allseg = __reduce_or_sync(0xffffffffu, (j == 0) ? segbits : 0u);
  return (phase_bits & ~allseg) | merged;
}

}  // namespace l3
