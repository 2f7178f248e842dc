// l3_decode_hwc.cuh — f3: the interleaved [H, W, 3] output ("HWC output (decode
// the 3 channel patches of a tile in one CTA)"). Included by l3_decode.cu after l3_decode_fast.cuh.
//
// The file stores the three channel planes of a patch as separate units, so an
// HWC element needs three independent bitstreams. One warp owns a TILE = (image, patch) for
// N <= 128 and decodes its R, G and B units in lock-step, each streamed through its own TMA ring
// (the same slot / mbarrier scheme as the planar kernel). After each row every lane holds 4
// columns x 3 channels and writes them as 12 contiguous bytes (u8: 3 x 32-bit stores) or 48 bytes
// (fp32: 3 x 128-bit stores) — full sectors, where the per-element strided stores of the augment
// variant touch a sector per 4-byte store. The row arithmetic (a3-a5) is decode_row, unchanged.
// Units with N > 128 go through the generic path (element stores, AUG layout bit).
#pragma once

namespace l3 {

constexpr int kHwcWarps = 2;
#ifndef L3_HWC_MIN_CTAS
#define L3_HWC_MIN_CTAS 8
#endif
#ifndef L3_HWC_SLOTS
#define L3_HWC_SLOTS 4
#endif
constexpr int kHwcSlots = L3_HWC_SLOTS;                       // 4 KB ring per channel stream
#ifndef L3_HWC_KTAB
#define L3_HWC_KTAB 1   // streamed tiles: a copy of the per-k unpack table after each channel ring (KT)
#endif
constexpr int kHwcKtab = kHwcSlots * kSlotBytes + 64;        // the table's offset in a channel ring region
constexpr int kHwcPitch = kHwcSlots * kSlotBytes + 64 + (L3_HWC_KTAB ? 256 : 0);   // + wrap mirror + table
// 3 rings per warp: 2 warps = 25 KB per CTA; the register file then bounds residency (16 warps / SM)
__host__ __device__ constexpr size_t hwc_smem_bytes() {
  return (size_t)kHwcWarps * 3 * kHwcPitch + (size_t)kHwcWarps * 3 * kHwcSlots * 8 + 16;
}

// Store modes of the interleaved epilogue.
constexpr int kStAligned = 0;   // every row start aligned (u8: 4 B, fp32: 16 B): 3 vector stores
constexpr int kStDynamic = 1;   // rows of varying alignment (image width not a multiple of 4)
constexpr int kStRagged = 2;    // the patch width is not a multiple of 4: per-column tests
constexpr int kStWindow = 3;    // crop window (f3): per-pixel validity mask, flip, any alignment

// Crop window of a tile (kStWindow): window row of the tile's current row, window height, which of
// the lane's 4 output pixels are inside the window and the patch, and the PRMT selector putting the
// lane's 4 pixels in output order (flip: reversed).
struct WinRow {
  int32_t ri;
  uint32_t chh, cmask, qsel;
};

// Row of a tile into a crop window, interleaved: the lane's 4 pixels x 3 channels in output order
// are 12 contiguous elements at optr; whole-lane pixels take the widest store the row's alignment
// allows (uniform across the warp: lanes differ by 12 / 48 bytes), lanes cut by the window or the
// patch edge store their valid pixels element by element.
template <bool F32>
__device__ __forceinline__ void store12w(uint8_t* optr, const LaneRows& r, const LaneRows& g, const LaneRows& b,
                                         const float* sc, const float* bi, bool live, const WinRow& wr) {
  if (!live || (uint32_t)wr.ri >= wr.chh || wr.cmask == 0u) return;
  const uint32_t qr = prmt(prmt(r.A, r.B, 0x6420u), 0u, wr.qsel);   // [R0 R1 R2 R3] in output order
  const uint32_t qg = prmt(prmt(g.A, g.B, 0x6420u), 0u, wr.qsel);
  const uint32_t qb = prmt(prmt(b.A, b.B, 0x6420u), 0u, wr.qsel);
  if (F32) {
    float v[12];
#pragma unroll
    for (int t = 0; t < 4; t++) {
      v[3 * t] = fmaf((float)((qr >> (8 * t)) & 0xFFu), sc[0], bi[0]);
      v[3 * t + 1] = fmaf((float)((qg >> (8 * t)) & 0xFFu), sc[1], bi[1]);
      v[3 * t + 2] = fmaf((float)((qb >> (8 * t)) & 0xFFu), sc[2], bi[2]);
    }
    float* o = reinterpret_cast<float*>(optr);
    if (wr.cmask == 0xFu) {
      if ((reinterpret_cast<uintptr_t>(optr) & 15u) == 0) {
#pragma unroll
        for (int q = 0; q < 3; q++)
          reinterpret_cast<float4*>(o)[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
      } else if ((reinterpret_cast<uintptr_t>(optr) & 7u) == 0) {
#pragma unroll
        for (int q = 0; q < 6; q++) reinterpret_cast<float2*>(o)[q] = make_float2(v[2 * q], v[2 * q + 1]);
      } else {
#pragma unroll
        for (int e = 0; e < 12; e++) o[e] = v[e];
      }
    } else {
#pragma unroll
      for (int t = 0; t < 4; t++)
        if ((wr.cmask >> t) & 1u) {
          o[3 * t] = v[3 * t];
          o[3 * t + 1] = v[3 * t + 1];
          o[3 * t + 2] = v[3 * t + 2];
        }
    }
  } else {
    const uint32_t x = prmt(qr, qg, 0x5140u);                    // R0 G0 R1 G1
    const uint32_t y = prmt(qr, qg, 0x7362u);                    // R2 G2 R3 G3
    const uint32_t w0 = prmt(x, qb, 0x2410u);                    // R0 G0 B0 R1
    const uint32_t w1 = prmt(prmt(x, qb, 0x0053u), y, 0x5410u);  // G1 B1 R2 G2
    const uint32_t w2 = prmt(y, qb, 0x7326u);                    // B2 R3 G3 B3
    const uint32_t wv[3] = {w0, w1, w2};
    if (wr.cmask == 0xFu) {
      if ((reinterpret_cast<uintptr_t>(optr) & 3u) == 0) {
#pragma unroll
        for (int q = 0; q < 3; q++) reinterpret_cast<uint32_t*>(optr)[q] = wv[q];
      } else if ((reinterpret_cast<uintptr_t>(optr) & 1u) == 0) {
#pragma unroll
        for (int q = 0; q < 6; q++)
          reinterpret_cast<uint16_t*>(optr)[q] = (uint16_t)(wv[q >> 1] >> (16 * (q & 1)));
      } else {
#pragma unroll
        for (int e = 0; e < 12; e++) optr[e] = (uint8_t)(wv[e >> 2] >> (8 * (e & 3)));
      }
    } else {
#pragma unroll
      for (int e = 0; e < 12; e++)
        if ((wr.cmask >> (e / 3)) & 1u) optr[e] = (uint8_t)(wv[e >> 2] >> (8 * (e & 3)));
    }
  }
}

// Row r of a tile, 4 columns of this lane, interleaved: R0 G0 B0 R1 G1 B1 R2 G2 B2 R3 G3 B3.
// r/g/b hold the row in pair form (A = columns 0, 1; B = columns 2, 3). kStDynamic picks the widest
// store the row's alignment allows; it is uniform across the warp (lanes differ by 12 or 48 bytes).
template <bool F32, int MODE>
__device__ __forceinline__ void store12(uint8_t* optr, const LaneRows& r, const LaneRows& g, const LaneRows& b,
                                        const float* sc, const float* bi, bool pred) {
  if (F32) {
    const uint32_t x[3][2] = {{r.A, r.B}, {g.A, g.B}, {b.A, b.B}};
    float v[12];
#pragma unroll
    for (int t = 0; t < 4; t++)
#pragma unroll
      for (int c = 0; c < 3; c++) {
        const uint32_t pr = x[c][t >> 1];
        // the low byte of each half (the pair may hold biased halves 0x6400 | c, L3_H2_HWC)
        v[3 * t + c] = fmaf((float)((t & 1) ? ((pr >> 16) & 0xFFu) : (pr & 0xFFu)), sc[c], bi[c]);
      }
    if (MODE == kStAligned) {
#pragma unroll
      for (int q = 0; q < 3; q++)
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %5, 0;\n\t"
            "@p st.global.v4.f32 [%0], {%1, %2, %3, %4};\n\t}" ::"l"(optr + 16 * q),
            "f"(v[4 * q]), "f"(v[4 * q + 1]), "f"(v[4 * q + 2]), "f"(v[4 * q + 3]), "r"((uint32_t)pred));
    } else if (pred) {
      float* o = reinterpret_cast<float*>(optr);
      if (MODE == kStRagged) {
#pragma unroll
        for (int t = 0; t < 4; t++)
          if (r.j4 + t < r.w) {
            o[3 * t] = v[3 * t];
            o[3 * t + 1] = v[3 * t + 1];
            o[3 * t + 2] = v[3 * t + 2];
          }
      } else if ((reinterpret_cast<uintptr_t>(optr) & 15u) == 0) {
#pragma unroll
        for (int q = 0; q < 3; q++)
          reinterpret_cast<float4*>(o)[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
      } else if ((reinterpret_cast<uintptr_t>(optr) & 7u) == 0) {
#pragma unroll
        for (int q = 0; q < 6; q++) reinterpret_cast<float2*>(o)[q] = make_float2(v[2 * q], v[2 * q + 1]);
      } else {
#pragma unroll
        for (int e = 0; e < 12; e++) o[e] = v[e];
      }
    }
  } else {
    const uint32_t x = prmt(r.A, g.A, 0x6240);   // R0 G0 R1 G1
    const uint32_t y = prmt(r.B, g.B, 0x6240);   // R2 G2 R3 G3
    const uint32_t z = prmt(b.A, b.B, 0x6420);   // B0 B1 B2 B3
    const uint32_t w0 = prmt(x, z, 0x2410);      // R0 G0 B0 R1
    const uint32_t w1 = prmt(prmt(x, z, 0x0053), y, 0x5410);   // G1 B1 R2 G2
    const uint32_t w2 = prmt(y, z, 0x7326);      // B2 R3 G3 B3
    if (MODE == kStAligned) {
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "@p st.global.b32 [%0], %1;\n\t@p st.global.b32 [%0+4], %2;\n\t@p st.global.b32 [%0+8], %3;\n\t}" ::"l"(
              optr),
          "r"(w0), "r"(w1), "r"(w2), "r"((uint32_t)pred));
    } else if (pred) {
      const uint32_t wv[3] = {w0, w1, w2};
      if (MODE == kStRagged) {
#pragma unroll
        for (int e = 0; e < 12; e++)
          if (r.j4 + e / 3 < r.w) optr[e] = (uint8_t)(wv[e >> 2] >> (8 * (e & 3)));
      } else if ((reinterpret_cast<uintptr_t>(optr) & 3u) == 0) {
#pragma unroll
        for (int q = 0; q < 3; q++) reinterpret_cast<uint32_t*>(optr)[q] = wv[q];
      } else if ((reinterpret_cast<uintptr_t>(optr) & 1u) == 0) {
#pragma unroll
        for (int q = 0; q < 6; q++)
          reinterpret_cast<uint16_t*>(optr)[q] = (uint16_t)(wv[q >> 1] >> (16 * (q & 1)));
      } else {
#pragma unroll
        for (int e = 0; e < 12; e++) optr[e] = (uint8_t)(wv[e >> 2] >> (8 * (e & 3)));
      }
    }
  }
}

// The rows of one tile: per row, the three channels' ring tests (STREAM), decode_row x 3, one
// interleaved store. Whole-staged tasks (!STREAM, N <= 32) run L-lane segments (GUARD).
template <bool F32, int MODE, bool STREAM>
__device__ __forceinline__ void hwc_tile_rows(LaneRows* s, uint8_t* rings, uint64_t* bars, StreamState* st,
                                              uint32_t* ph, uint32_t h, uint8_t* optr, uint32_t pitch,
                                              const float* sc, const float* bi, uint32_t K, const uint8_t* src,
                                              uint64_t lim, int lane, uint32_t Lw, bool valid, WinRow wr = {}) {
  constexpr bool FAST = MODE != kStRagged && MODE != kStWindow;   // window tiles may be ragged: ghost columns
  constexpr bool GUARD = !STREAM;
  constexpr int SLOTS = STREAM ? kHwcSlots : 16;   // whole-staged: one linear 12 KB buffer, no wrap
  // streamed: the unpack table copy after each channel ring (rewritten per tile: whole-staged tasks may
  // have staged over it); whole-staged: the static table
  constexpr int KT = (STREAM && L3_HWC_KTAB) ? kHwcKtab : 0;
  constexpr uint32_t rowmax = (12u + 8u * 128u) / 8u + 10u;
#pragma unroll
  for (int c = 0; c < 3; c++) {
    uint8_t* ring = STREAM ? rings + c * kHwcPitch : rings;
    if (STREAM && (s[c].bp >> 3) + 2u * rowmax > st[c].landed_end)
      stream_advance<kHwcSlots>(src, lim, st[c], ring, bars + c * kHwcSlots, ph[c], s[c].bp >> 3,
                                (s[c].bp >> 3) + 2u * rowmax, lane);
    s[c].raw = rbits<SLOTS>(ring, s[c].bp);
  }
#pragma unroll
  for (int c = 0; c < 3; c++)
    decode_row<true, false, FAST, GUARD, false, false, SLOTS, false, !FAST, 0, KT>(
        s[c], STREAM ? rings + c * kHwcPitch : rings, 0, Lw, 0.f, 0.f, K);
  if (MODE == kStWindow) store12w<F32>(optr, s[0], s[1], s[2], sc, bi, s[0].h > 0, wr);
  else store12<F32, MODE>(optr, s[0], s[1], s[2], sc, bi, valid && s[0].h > 0);
  optr += pitch;
  wr.ri++;
  for (uint32_t r = 1; r < h; r++) {
    if (STREAM) {
#pragma unroll
      for (int c = 0; c < 3; c++) {
        if ((s[c].bp >> 3) + rowmax > st[c].landed_end)
          stream_advance<kHwcSlots>(src, lim, st[c], rings + c * kHwcPitch, bars + c * kHwcSlots, ph[c],
                                    s[c].bp >> 3, (s[c].bp >> 3) + 2u * rowmax, lane);
      }
    }
#pragma unroll
    for (int c = 0; c < 3; c++)
      decode_row<false, false, FAST, GUARD, false, false, SLOTS, false, !FAST, 0, KT>(
          s[c], STREAM ? rings + c * kHwcPitch : rings, r, Lw, 0.f, 0.f, K);
    if (MODE == kStWindow) store12w<F32>(optr, s[0], s[1], s[2], sc, bi, r < s[0].h, wr);
    else store12<F32, MODE>(optr, s[0], s[1], s[2], sc, bi, valid && r < s[0].h);
    optr += pitch;
    wr.ri++;
  }
}

// Output of a tile into the crop window of image d (f3, kStWindow): the lane's lowest-address pixel,
// the row pitch, and the window row / validity / order of the lane's pixels. Every row of the tile
// from its top is decoded (the row dependency); rows outside the window store nothing.
template <bool F32>
__device__ __forceinline__ uint8_t* hwc_window(const DecodeParams& p, const ImgDesc& d, uint32_t x0, uint32_t y0,
                                               uint32_t w, uint32_t j4, bool act, WinRow& wr, uint32_t& pitch) {
  const uint32_t esz = F32 ? 4u : 1u;
  const bool flip = (d.flip & 1u) != 0;
  const int32_t cw = (int32_t)d.cw, cj0 = (int32_t)(x0 + j4) - (int32_t)d.cx;
  const int32_t bc = flip ? cw - 4 - cj0 : cj0;   // window column of the lane's lowest-address pixel
  wr.ri = (int32_t)y0 - (int32_t)d.cy;
  wr.chh = d.ch;
  wr.qsel = flip ? 0x0123u : 0x3210u;
  wr.cmask = 0;
#pragma unroll
  for (int t = 0; t < 4; t++) {
    const int32_t c = flip ? 3 - t : t;
    if (act && j4 + (uint32_t)c < w && cj0 + c >= 0 && cj0 + c < cw) wr.cmask |= 1u << t;
  }
  pitch = (uint32_t)cw * 3u * esz;
  return reinterpret_cast<uint8_t*>(p.out) + (int64_t)d.out_off * esz + ((int64_t)wr.ri * cw + bc) * 3 * (int64_t)esz;
}

// N <= 32 (mode 6): G = 32 / L tiles per task, one L-lane segment each (as mode 0 of the planar
// kernel). The task's 3G units are staged whole into the warp's 12 KB buffer with one barrier;
// if they do not fit (near-incompressible content), the tiles are staged and decoded one per pass.
template <bool F32, bool WIN>
__device__ __forceinline__ uint32_t hwc_small_task(const DecodeParams& p, const ImgDesc& d, int img, uint32_t t,
                                                   uint8_t* buf, uint64_t* bars, uint32_t ph0, uint64_t lim,
                                                   uint32_t K, int lane) {
  constexpr uint32_t kCap = 3u * kHwcPitch - 64u;   // staging capacity (keeps the 8-byte reads in bounds)
  const uint32_t esz = F32 ? 4u : 1u;
  const uint32_t L = d.L, G = d.G;
  const uint32_t seg = (uint32_t)lane / L, j = (uint32_t)lane % L;
  constexpr bool crop = WIN;        // f3 crop window (the kernel instantiation with windows)
  const uint32_t v = t * G + seg;   // tile of the task's image (crop: among the window's tiles)
  const bool tact = v < (crop ? d.gxw * d.gyw : d.P);
  const uint32_t tile = crop ? (d.py0 + v / d.gxw) * d.gx + d.px0 + v % d.gxw : v;
  uint32_t x0 = 0, y0 = 0, w = 0, h = 0;
  if (tact) {
    x0 = (tile % d.gx) * d.N;
    y0 = (tile / d.gx) * d.N;
    w = min(d.N, d.W - x0);
    h = min(d.N, d.H - y0);
    if (crop) h = min(h, d.cy + d.ch - y0);   // rows below the window are not needed
  }
  const uint32_t nunits = 3u * d.P;
  const uint8_t* file = p.pp.src + d.file_off;
  const uint32_t worst = worst_patch_bytes(w, h);
  uint64_t start[3], end[3], a16[3], sEnd[3];
  uint32_t bytes[3], len[3];
  bool act[3];
  uint32_t total = 0;
#pragma unroll
  for (int c = 0; c < 3; c++) {
    const uint32_t u = (uint32_t)c * d.P + tile;
    uint64_t off = 0, nxt = 0;
    if (tact) {
      off = ld_u32le(file + 13 + 4ull * u);
      nxt = (u + 1 < nunits) ? (uint64_t)ld_u32le(file + 17 + 4ull * u) : d.data_len;
    }
    act[c] = tact && !(unit_offsets_bad(u, nunits, off, nxt, d.data_len));
    if (tact && !act[c] && j == 0) record_err(&p.pp.ws.errkey[img], 0u);   // header-level: CORRUPT_HEADER
    start[c] = act[c] ? d.data_off + off : 0;
    end[c] = act[c] ? d.data_off + nxt : 0;
    sEnd[c] = act[c] ? min(end[c], start[c] + worst + 8) : 0;
    a16[c] = start[c] & ~15ull;
    bytes[c] = act[c] ? (uint32_t)(((sEnd[c] + 15) & ~15ull) - a16[c]) : 0u;
    len[c] = act[c] ? (uint32_t)min((uint64_t)(worst + 16), end[c] - start[c]) : 0u;
    total += bytes[c];
  }
  // one pass if the task's units fit the buffer, else one tile per pass
  uint32_t incl = (j == 0) ? total : 0u;   // inclusive scan over the segments (leader lanes)
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  const uint32_t sum = __shfl_sync(0xffffffffu, incl, 31);
  const uint32_t seg_excl = __shfl_sync(0xffffffffu, incl, seg * L) - __shfl_sync(0xffffffffu, (j == 0) ? total : 0u,
                                                                                   seg * L);
  const bool one = sum <= kCap;
  const uint32_t npass = one ? 1u : G;
  const float sc[3] = {F32 ? p.scale[0] : 0.f, F32 ? p.scale[1] : 0.f, F32 ? p.scale[2] : 0.f};
  const float bi[3] = {F32 ? p.bias[0] : 0.f, F32 ? p.bias[1] : 0.f, F32 ? p.bias[2] : 0.f};
  const uint32_t pitch = d.W * 3u * esz;
  for (uint32_t q = 0; q < npass; q++) {
    const bool mine = tact && (one || seg == q);
    const uint32_t base = one ? seg_excl : 0u;
    // a2: stage this pass's units (bulk copies on bars[0], < 16 tail bytes past `lim` by the lanes)
    uint32_t bulk[3], off_c[3];
    uint32_t tx = 0, cum = 0;
#pragma unroll
    for (int c = 0; c < 3; c++) {
      off_c[c] = base + cum;
      cum += bytes[c];
      const uint64_t b16 = a16[c] + bytes[c];
      const uint64_t be = b16 < lim ? b16 : lim;
      bulk[c] = (mine && be > a16[c]) ? (uint32_t)(be - a16[c]) : 0u;
      tx += bulk[c];
    }
    uint32_t txw = (mine && j == 0) ? tx : 0u;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) txw += __shfl_xor_sync(0xffffffffu, txw, o);
    if (lane == 0) mbar_arrive_expect_tx(&bars[0], txw);
    __syncwarp();
    if (mine) {
#pragma unroll
      for (int c = 0; c < 3; c++) {
        uint8_t* dst = buf + off_c[c];
        if (j == 0 && bulk[c]) bulk_g2s(dst, p.pp.src + a16[c], bulk[c], &bars[0]);
        const uint64_t b16 = a16[c] + bytes[c];
        const uint64_t t0 = a16[c] > lim ? a16[c] : lim;
        for (uint64_t x = t0 + j; x < sEnd[c] && x < b16; x += L) dst[x - a16[c]] = __ldg(p.pp.src + x);
      }
    }
    mbar_wait(&bars[0], ph0 & 1u);
    ph0 ^= 1u;
    __syncwarp();
    if (mine) {
#pragma unroll
      for (int c = 0; c < 3; c++) swap_words(buf + off_c[c], 0, bytes[c], j, L);
    }
    __syncwarp();
    // a3-a6
    LaneRows s[3];
#pragma unroll
    for (int c = 0; c < 3; c++) {
      s[c].w = w;
      s[c].h = (mine && act[c]) ? h : 0u;
      s[c].j4 = 4u * j;
      s[c].first = (j == 0);
      s[c].last = (s[c].j4 + 4u >= w);
      s[c].valid = mine && s[c].j4 < w;
      s[c].kacc = 0;
      s[c].A = s[c].B = 0;
      s[c].bp = (off_c[c] + (uint32_t)(start[c] - a16[c])) * 8u;
      s[c].lim = s[c].bp + len[c] * 8u;
    }
    uint32_t hmax = mine ? h : 0u;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) hmax = max(hmax, __shfl_xor_sync(0xffffffffu, hmax, o));
    uint8_t* optr = reinterpret_cast<uint8_t*>(p.out) + (d.out_off + ((uint64_t)y0 * d.W + x0 + 4u * j) * 3u) * esz;
    const bool ragged = __any_sync(0xffffffffu, mine && (w & 3u) != 0);
    const bool aligned = __all_sync(0xffffffffu, !mine || ((reinterpret_cast<uintptr_t>(optr) & (F32 ? 15 : 3)) == 0 &&
                                                          (pitch & (F32 ? 15u : 3u)) == 0));
    const bool valid = s[0].valid && s[1].h > 0 && s[2].h > 0;
    StreamState* nost = nullptr;
    if constexpr (crop) {   // f3: crop window (any alignment, flip, partial lanes)
      WinRow wr;
      uint32_t wpitch;
      uint8_t* wptr = hwc_window<F32>(p, d, x0, y0, w, 4u * j, mine && act[0] && act[1] && act[2], wr, wpitch);
      if (hmax > 0)
        hwc_tile_rows<F32, kStWindow, false>(s, buf, bars, nost, nullptr, hmax, wptr, wpitch, sc, bi, K, p.pp.src,
                                             lim, lane, L, valid, wr);
    } else if (hmax > 0) {
      if (ragged)
        hwc_tile_rows<F32, kStRagged, false>(s, buf, bars, nost, nullptr, hmax, optr, pitch, sc, bi, K, p.pp.src,
                                             lim, lane, L, valid);
      else if (aligned)
        hwc_tile_rows<F32, kStAligned, false>(s, buf, bars, nost, nullptr, hmax, optr, pitch, sc, bi, K, p.pp.src,
                                              lim, lane, L, valid);
      else
        hwc_tile_rows<F32, kStDynamic, false>(s, buf, bars, nost, nullptr, hmax, optr, pitch, sc, bi, K, p.pp.src,
                                              lim, lane, L, valid);
    }
#pragma unroll
    for (int c = 0; c < 3; c++) {
      const bool err = mine && act[c] && (s[c].kacc >= 0x80000000u || s[c].bp > s[c].lim);
      if (err && j == 0) {   // a7: exact first error of a failed unit
        const int code = unit_first_error(p.pp.src, start[c], end[c], w, h);
        if (code != L3_OK) record_err(&p.pp.ws.errkey[img], err_key((uint32_t)c * d.P + tile, code));
      }
    }
    __syncwarp();
    fence_proxy_async_smem();
  }
  return ph0;
}

// WIN: crop windows (f3); a separate instantiation, so the full-image kernel's registers are untouched.
template <bool F32, bool WIN>
__global__ void __launch_bounds__(kHwcWarps * 32, L3_HWC_MIN_CTAS) l3_decode_hwc_kernel(DecodeParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ unsigned int ticket;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* rings = smem + warp * 3 * kHwcPitch;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kHwcWarps * 3 * kHwcPitch) + warp * 3 * kHwcSlots;
  if (lane == 0) {
    for (int s = 0; s < 3 * kHwcSlots; s++) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  if (L3_UNPACK_TAB) {
    init_ktab();
    __syncthreads();
  }
  __syncwarp();
  uint32_t ph[3] = {0u, 0u, 0u};
  WsHead* head = p.pp.ws.head;

  // a1 ran in the preceding l3_prep_kernel (PDL; tasks = tiles for N <= 128)
  pdl_wait();

  const uint64_t* prefix = p.pp.ws.prefix[0];
  const uint64_t total_tasks = prefix[p.pp.n];
  const uint64_t lim = p.pp.src_offsets[p.pp.n] & ~15ull;
  const uint32_t K = p.key_scale;
  const uint32_t esz = F32 ? 4u : 1u;

  const uint64_t grid_warps = (uint64_t)gridDim.x * kHwcWarps;   // first task: the grid-wide warp index
  uint64_t task = (uint64_t)blockIdx.x * kHwcWarps + warp;
  while (task < total_tasks) {
    int lo = 0, hi = p.pp.n;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (__ldcg(&prefix[mid]) <= task) lo = mid; else hi = mid;
    }
    const int img = lo;
    const ImgDesc d = p.pp.ws.desc[img];
    const uint32_t pp = (uint32_t)(task - prefix[img]);   // patch index: the tile (mode 6: tile group)
    uint64_t next = 0;
    if (lane == 0) next = grid_warps + atomicAdd(&head->next_task[0], 1ull);
    if (d.mode == 6) {   // N <= 32: G tiles per task, whole-staged
      ph[0] = hwc_small_task<F32, WIN>(p, d, img, pp, rings, bars, ph[0], lim, K, lane);
      task = __shfl_sync(0xffffffffu, next, 0);
      continue;
    }

    constexpr bool crop = WIN;   // f3: pp counts the window's tiles
    const uint32_t px = crop ? d.px0 + pp % d.gxw : pp % d.gx, py = crop ? d.py0 + pp / d.gxw : pp / d.gx;
    const uint32_t tile = py * d.gx + px;
    const uint32_t x0 = px * d.N, y0 = py * d.N;
    const uint32_t w = min(d.N, d.W - x0);
    const uint32_t h = crop ? min(min(d.N, d.H - y0), d.cy + d.ch - y0) : min(d.N, d.H - y0);
    const uint32_t nunits = 3u * d.P;
    const uint8_t* file = p.pp.src + d.file_off;
    const uint32_t worst = worst_patch_bytes(w, h);

    LaneRows s[3];
    StreamState st[3];
    uint64_t start[3], end[3];
    bool act[3];
#pragma unroll
    for (int c = 0; c < 3; c++) {
      const uint32_t u = (uint32_t)c * d.P + tile;
      const uint64_t off = ld_u32le(file + 13 + 4ull * u);
      const uint64_t nxt = (u + 1 < nunits) ? (uint64_t)ld_u32le(file + 17 + 4ull * u) : d.data_len;
      act[c] = !(unit_offsets_bad(u, nunits, off, nxt, d.data_len));
      if (!act[c] && lane == 0) record_err(&p.pp.ws.errkey[img], 0u);   // header-level: CORRUPT_HEADER
      start[c] = act[c] ? d.data_off + off : 0;
      end[c] = act[c] ? d.data_off + nxt : 0;
      const uint64_t stage_end = act[c] ? min(end[c], start[c] + worst + 8) : 0;
      const uint32_t len = act[c] ? (uint32_t)min((uint64_t)(worst + 16), end[c] - start[c]) : 0u;
      s[c].w = w;
      s[c].h = act[c] ? h : 0u;
      s[c].j4 = 4u * lane;
      s[c].first = (lane == 0);
      s[c].last = (s[c].j4 + 4u >= w);
      s[c].valid = s[c].j4 < w;
      s[c].kacc = 0;
      s[c].A = s[c].B = 0;
      st[c].A = start[c] & ~15ull;
      st[c].B = (stage_end + 15) & ~15ull;
      st[c].stage_end = stage_end;
      stream_rel_init(st[c], lim);
      st[c].nchunks = act[c] ? (uint32_t)((st[c].B - st[c].A + kSlotBytes - 1) / kSlotBytes) : 0u;
      st[c].issued = 0;
      st[c].landed = 0;
      st[c].landed_end = 0;
      const uint32_t first = min(st[c].nchunks, (uint32_t)kHwcSlots);
      while (st[c].issued < first)
        stream_issue<kHwcSlots>(p.pp.src, lim, st[c], rings + c * kHwcPitch, bars + c * kHwcSlots, lane);
      s[c].bp = act[c] ? (uint32_t)(start[c] - st[c].A) * 8u : 0u;
      s[c].lim = s[c].bp + len * 8u;
    }
    if (L3_HWC_KTAB && lane < 16) {   // the unpack table after each channel ring (see hwc_tile_rows)
      const uint32_t k = (uint32_t)lane;
      const uint4 e = (k >= 1 && k <= 8) ? make_uint4(32u - k, 16u - 2u * k, 2u * k, ((1u << k) - 1u) << 16)
                                         : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
      for (int c = 0; c < 3; c++) reinterpret_cast<uint4*>(rings + c * kHwcPitch + kHwcKtab)[k] = e;
    }
    __syncwarp();

    // output: element (y0 + r, x0 + j4, 0) of the image's [H, W, 3] block
    const uint32_t pitch = d.W * 3u * esz;
    uint8_t* optr = reinterpret_cast<uint8_t*>(p.out) +
                    (d.out_off + ((uint64_t)y0 * d.W + x0 + 4u * lane) * 3u) * esz;
    const bool aligned = (reinterpret_cast<uintptr_t>(optr) & (F32 ? 15 : 3)) == 0 && (pitch & (F32 ? 15u : 3u)) == 0;
    const bool ragged = (w & 3u) != 0;   // warp-uniform: one tile per warp
    const bool aligned_all = __all_sync(0xffffffffu, aligned);
    const float sc[3] = {F32 ? p.scale[0] : 0.f, F32 ? p.scale[1] : 0.f, F32 ? p.scale[2] : 0.f};
    const float bi[3] = {F32 ? p.bias[0] : 0.f, F32 ? p.bias[1] : 0.f, F32 ? p.bias[2] : 0.f};
    const bool valid = s[0].valid;
    if constexpr (crop) {   // f3: crop window (any alignment, flip, partial lanes)
      WinRow wr;
      uint32_t wpitch;
      uint8_t* wptr = hwc_window<F32>(p, d, x0, y0, w, 4u * lane, act[0] && act[1] && act[2], wr, wpitch);
      hwc_tile_rows<F32, kStWindow, true>(s, rings, bars, st, ph, h, wptr, wpitch, sc, bi, K, p.pp.src, lim, lane,
                                          32u, valid, wr);
    } else if (ragged)
      hwc_tile_rows<F32, kStRagged, true>(s, rings, bars, st, ph, h, optr, pitch, sc, bi, K, p.pp.src, lim, lane,
                                          32u, valid);
    else if (aligned_all)
      hwc_tile_rows<F32, kStAligned, true>(s, rings, bars, st, ph, h, optr, pitch, sc, bi, K, p.pp.src, lim, lane,
                                           32u, valid);
    else
      hwc_tile_rows<F32, kStDynamic, true>(s, rings, bars, st, ph, h, optr, pitch, sc, bi, K, p.pp.src, lim, lane,
                                           32u, valid);

#pragma unroll
    for (int c = 0; c < 3; c++) {
      const bool err = act[c] && (s[c].kacc >= 0x80000000u || s[c].bp > s[c].lim);
      if (err && lane == 0) {   // a7: exact first error of a failed unit
        const int code = unit_first_error(p.pp.src, start[c], end[c], w, h);
        if (code != L3_OK) record_err(&p.pp.ws.errkey[img], err_key((uint32_t)c * d.P + tile, code));
      }
      while (st[c].landed < st[c].issued) {   // drain copies that were issued but never waited for
        const uint32_t sl = st[c].landed % kHwcSlots;
        mbar_wait(&bars[c * kHwcSlots + sl], (ph[c] >> sl) & 1u);
        ph[c] ^= 1u << sl;
        st[c].landed++;
      }
    }
    __syncwarp();
    fence_proxy_async_smem();
    task = __shfl_sync(0xffffffffu, next, 0);
  }

  // N > 128 units: generic path (element stores in the HWC layout, ImgDesc.flip bit 1)
  const uint64_t total1 = p.pp.ws.prefix[1][p.pp.n];
  if (total1 > 0) {
    GenericArgs ga;
    ga.src = p.pp.src;
    ga.prefix1 = p.pp.ws.prefix[1];
    ga.desc = p.pp.ws.desc;
    ga.a1_pre1 = nullptr;
    ga.a1_desc = nullptr;
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
      // the generic path's 8 KB ring / 8 barriers = rings 0 and 1 with their 4 + 4 barriers
      uint32_t gp = (ph[0] & 0xFu) | ((ph[1] & 0xFu) << 4);
      gp = generic_task<F32, true, true>(ga, t1, rings, bars, gp);
      ph[0] = gp & 0xFu;
      ph[1] = (gp >> 4) & 0xFu;
    }
  }

  // a7: per-image status by the last CTA, which also re-zeroes the workspace head
  a7_finish(p.pp, head, &ticket);
}

}  // namespace l3
