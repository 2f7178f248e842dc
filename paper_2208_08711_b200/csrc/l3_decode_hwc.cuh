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
constexpr int kHwcPitch = kHwcSlots * kSlotBytes + 64;        // + wrap mirror
// 3 rings per warp: 2 warps = 25 KB per CTA; the register file then bounds residency (16 warps / SM)
__host__ __device__ constexpr size_t hwc_smem_bytes() {
  return (size_t)kHwcWarps * 3 * kHwcPitch + (size_t)kHwcWarps * 3 * kHwcSlots * 8 + 16;
}

// Row r of a tile, 4 columns of this lane, interleaved: R0 G0 B0 R1 G1 B1 R2 G2 B2 R3 G3 B3.
// r/g/b hold the row in pair form (A = columns 0, 1; B = columns 2, 3).
template <bool F32, bool FAST>
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
        v[3 * t + c] = fmaf((float)((t & 1) ? (pr >> 16) : (pr & 0xFFFFu)), sc[c], bi[c]);
      }
    if (FAST) {
#pragma unroll
      for (int q = 0; q < 3; q++)
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %5, 0;\n\t"
            "@p st.global.v4.f32 [%0], {%1, %2, %3, %4};\n\t}" ::"l"(optr + 16 * q),
            "f"(v[4 * q]), "f"(v[4 * q + 1]), "f"(v[4 * q + 2]), "f"(v[4 * q + 3]), "r"((uint32_t)pred));
    } else if (pred) {
      float* o = reinterpret_cast<float*>(optr);
#pragma unroll
      for (int t = 0; t < 4; t++)
        if (r.j4 + t < r.w) {
          o[3 * t] = v[3 * t];
          o[3 * t + 1] = v[3 * t + 1];
          o[3 * t + 2] = v[3 * t + 2];
        }
    }
  } else {
    const uint32_t x = prmt(r.A, g.A, 0x6240);   // R0 G0 R1 G1
    const uint32_t y = prmt(r.B, g.B, 0x6240);   // R2 G2 R3 G3
    const uint32_t z = prmt(b.A, b.B, 0x6420);   // B0 B1 B2 B3
    const uint32_t w0 = prmt(x, z, 0x2410);      // R0 G0 B0 R1
    const uint32_t w1 = prmt(prmt(x, z, 0x0053), y, 0x5410);   // G1 B1 R2 G2
    const uint32_t w2 = prmt(y, z, 0x7326);      // B2 R3 G3 B3
    if (FAST) {
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "@p st.global.b32 [%0], %1;\n\t@p st.global.b32 [%0+4], %2;\n\t@p st.global.b32 [%0+8], %3;\n\t}" ::"l"(
              optr),
          "r"(w0), "r"(w1), "r"(w2), "r"((uint32_t)pred));
    } else if (pred) {
      const uint32_t wv[3] = {w0, w1, w2};
#pragma unroll
      for (int e = 0; e < 12; e++)
        if (r.j4 + e / 3 < r.w) optr[e] = (uint8_t)(wv[e >> 2] >> (8 * (e & 3)));
    }
  }
}

// The rows of one tile: per row, the three channels' ring tests, decode_row x 3, one store.
template <bool F32, bool FAST>
__device__ __forceinline__ void hwc_tile_rows(LaneRows* s, uint8_t* rings, uint64_t* bars, StreamState* st,
                                              uint32_t* ph, uint32_t h, uint8_t* optr, uint32_t pitch,
                                              const float* sc, const float* bi, uint32_t K, const uint8_t* src,
                                              uint64_t lim, int lane) {
  constexpr uint32_t rowmax = (12u + 8u * 128u) / 8u + 10u;
#pragma unroll
  for (int c = 0; c < 3; c++) {
    uint8_t* ring = rings + c * kHwcPitch;
    if ((s[c].bp >> 3) + 2u * rowmax > st[c].landed_end)
      stream_advance<kHwcSlots>(src, lim, st[c], ring, bars + c * kHwcSlots, ph[c], s[c].bp >> 3,
                                (s[c].bp >> 3) + 2u * rowmax, lane);
    s[c].raw = rbits<kHwcSlots>(ring, s[c].bp);
  }
#pragma unroll
  for (int c = 0; c < 3; c++)
    decode_row<true, false, FAST, false, false, false, kHwcSlots>(s[c], rings + c * kHwcPitch, 0, 32u, 0.f, 0.f, K);
  store12<F32, FAST>(optr, s[0], s[1], s[2], sc, bi, s[0].valid);
  optr += pitch;
  for (uint32_t r = 1; r < h; r++) {
#pragma unroll
    for (int c = 0; c < 3; c++) {
      if ((s[c].bp >> 3) + rowmax > st[c].landed_end)
        stream_advance<kHwcSlots>(src, lim, st[c], rings + c * kHwcPitch, bars + c * kHwcSlots, ph[c],
                                  s[c].bp >> 3, (s[c].bp >> 3) + 2u * rowmax, lane);
    }
#pragma unroll
    for (int c = 0; c < 3; c++)
      decode_row<false, false, FAST, false, false, false, kHwcSlots>(s[c], rings + c * kHwcPitch, r, 32u, 0.f, 0.f,
                                                                     K);
    store12<F32, FAST>(optr, s[0], s[1], s[2], sc, bi, s[0].valid);
    optr += pitch;
  }
}

template <bool F32>
__global__ void __launch_bounds__(kHwcWarps * 32, L3_HWC_MIN_CTAS) l3_decode_hwc_kernel(DecodeParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t sh_a[33], sh_b[33];
  __shared__ unsigned int ticket;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* rings = smem + warp * 3 * kHwcPitch;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kHwcWarps * 3 * kHwcPitch) + warp * 3 * kHwcSlots;
  if (lane == 0) {
    for (int s = 0; s < 3 * kHwcSlots; s++) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncwarp();
  uint32_t ph[3] = {0u, 0u, 0u};
  WsHead* head = p.pp.ws.head;

  // a1 inside the launch (as in l3_decode_kernel): tasks = tiles for N <= 128
  if (blockIdx.x == 0) {
    parse_phase_simple<false, true, true>(p.pp, sh_a, sh_b);
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) st_release_gpu(&head->ready, 1u);
  } else {
    if (threadIdx.x == 0) {
      while (ld_acquire_gpu(&head->ready) == 0u) __nanosleep(64);
    }
    __syncthreads();
  }

  const uint64_t* prefix = p.pp.ws.prefix[0];
  const uint64_t total_tasks = prefix[p.pp.n];
  const uint64_t lim = p.pp.src_offsets[p.pp.n] & ~15ull;
  const uint32_t K = p.key_scale;
  const uint32_t esz = F32 ? 4u : 1u;

  uint64_t task = 0;
  if (lane == 0) task = atomicAdd(&head->next_task[0], 1ull);
  task = __shfl_sync(0xffffffffu, task, 0);
  while (task < total_tasks) {
    int lo = 0, hi = p.pp.n;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (__ldg(&prefix[mid]) <= task) lo = mid; else hi = mid;
    }
    const int img = lo;
    const ImgDesc d = p.pp.ws.desc[img];
    const uint32_t pp = (uint32_t)(task - prefix[img]);   // patch index: the tile
    uint64_t next = 0;
    if (lane == 0) next = atomicAdd(&head->next_task[0], 1ull);

    const uint32_t px = pp % d.gx, py = pp / d.gx;
    const uint32_t x0 = px * d.N, y0 = py * d.N;
    const uint32_t w = min(d.N, d.W - x0), h = min(d.N, d.H - y0);
    const uint32_t nunits = 3u * d.P;
    const uint8_t* file = p.pp.src + d.file_off;
    const uint32_t worst = worst_patch_bytes(w, h);

    LaneRows s[3];
    StreamState st[3];
    uint64_t start[3], end[3];
    bool act[3];
#pragma unroll
    for (int c = 0; c < 3; c++) {
      const uint32_t u = (uint32_t)c * d.P + pp;
      const uint64_t off = ld_u32le(file + 13 + 4ull * u);
      const uint64_t nxt = (u + 1 < nunits) ? (uint64_t)ld_u32le(file + 17 + 4ull * u) : d.data_len;
      act[c] = !((u == 0 && off != 0) || off >= d.data_len || (u + 1 < nunits && nxt <= off));
      if (!act[c] && lane == 0) atomicMin(&p.pp.ws.errkey[img], 0u);   // header-level: CORRUPT_HEADER
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
    __syncwarp();

    // output: element (y0 + r, x0 + j4, 0) of the image's [H, W, 3] block
    const uint32_t pitch = d.W * 3u * esz;
    uint8_t* optr = reinterpret_cast<uint8_t*>(p.out) +
                    (d.out_off + ((uint64_t)y0 * d.W + x0 + 4u * lane) * 3u) * esz;
    const bool fast_ok = (w & 3u) == 0 && (reinterpret_cast<uintptr_t>(optr) & (F32 ? 15 : 3)) == 0 &&
                         (pitch & (F32 ? 15u : 3u)) == 0;
    const bool fast = __all_sync(0xffffffffu, fast_ok);
    const float sc[3] = {F32 ? p.scale[0] : 0.f, F32 ? p.scale[1] : 0.f, F32 ? p.scale[2] : 0.f};
    const float bi[3] = {F32 ? p.bias[0] : 0.f, F32 ? p.bias[1] : 0.f, F32 ? p.bias[2] : 0.f};
    if (fast)
      hwc_tile_rows<F32, true>(s, rings, bars, st, ph, h, optr, pitch, sc, bi, K, p.pp.src, lim, lane);
    else
      hwc_tile_rows<F32, false>(s, rings, bars, st, ph, h, optr, pitch, sc, bi, K, p.pp.src, lim, lane);

#pragma unroll
    for (int c = 0; c < 3; c++) {
      const bool err = act[c] && (s[c].kacc >= 0x80000000u || s[c].bp > s[c].lim);
      if (err && lane == 0) {   // a7: exact first error of a failed unit
        const int code = unit_first_error(p.pp.src, start[c], end[c], w, h);
        if (code != L3_OK) atomicMin(&p.pp.ws.errkey[img], err_key((uint32_t)c * d.P + pp, code));
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
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    ticket = atomicAdd(&head->done_ctas, 1u);
  }
  __syncthreads();
  if (ticket == gridDim.x - 1) {
    __threadfence();
    for (int i = threadIdx.x; i < p.pp.n; i += blockDim.x) {
      if (p.pp.status[i] != L3_OK) continue;
      const uint32_t key = atomicAdd(&p.pp.ws.errkey[i], 0u);
      if (key == kNoError) continue;
      if (key == 0u) {
        p.pp.status[i] = L3_E_CORRUPT_HEADER;
      } else {
        p.pp.status[i] = (key & 1u) ? L3_E_TRUNCATED_STREAM : L3_E_CORRUPT_STREAM;
        if (p.pp.bad_unit) p.pp.bad_unit[i] = (int32_t)((key >> 1) & 0x3FFFFFFFu);
      }
    }
    if (threadIdx.x == 0) {
      head->next_task[0] = 0;
      head->next_task[1] = 0;
      head->done_ctas = 0;
      head->ready = 0;
    }
  }
}

}  // namespace l3
