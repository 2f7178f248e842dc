// l3_encode.cu — sm_100a batch ENCODER.
//
// Offline dataset conversion on the GPU, byte-identical to the oracle's CPU
// encoder under the same readings (C1 residual mod 256, C2 signed
// base for residual rows, C3 tie order, C4 clamp-to-edge, C5 first row per
// patch, C6 k >= 1, C8 MSB-first rows, byte-aligned patches, C9 container).
// Not on the decode hot path: one warp per (image, channel, patch) unit, 4
// consecutive columns per lane; each lane ORs its 4 deltas into the unit's
// shared-memory bitstream as one field (two word atomics per lane and row).
//
//   E1 l3_enc_size_kernel   bytes of every unit (two-pass: sizes first)
//   E2 l3_enc_scan_kernel   per image: unit offsets (exclusive scan) + file size
//   E3 l3_enc_files_kernel  file offsets across the batch (single CTA scan)
//   E4 l3_enc_pack_kernel   header + offset table + packed bitstream per unit
#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "l3_internal.cuh"

namespace l3 {

struct EncDesc {
  uint64_t img_off;     // byte offset of the planar image in `images`
  uint64_t unit0;       // global index of this image's first unit
  uint32_t W, H, N, gx, P;
  uint32_t hdr;         // 13 + 12P (fits: P bounded by the host check)
};

struct EncWs {
  EncDesc* desc;        // n
  uint64_t* unit_prefix;  // n+1 (global unit index)
  uint32_t* unit_bytes;   // total units
  uint32_t* unit_off;     // total units (relative to the data section)
  uint64_t* file_size;    // n
  static uint64_t bytes(int n, uint64_t units) {
    return align_up(sizeof(EncDesc) * (uint64_t)n, 256) + align_up(8ull * (n + 1), 256) +
           2 * align_up(4ull * units, 256) + align_up(8ull * n, 256);
  }
  static EncWs at(void* ws, int n, uint64_t units) {
    EncWs v;
    char* p = (char*)ws;
    v.desc = (EncDesc*)p; p += align_up(sizeof(EncDesc) * (uint64_t)n, 256);
    v.unit_prefix = (uint64_t*)p; p += align_up(8ull * (n + 1), 256);
    v.unit_bytes = (uint32_t*)p; p += align_up(4ull * units, 256);
    v.unit_off = (uint32_t*)p; p += align_up(4ull * units, 256);
    v.file_size = (uint64_t*)p;
    return v;
  }
};

struct EncParams {
  const uint8_t* images;
  int n;
  uint64_t total_units;
  uint8_t* dst;
  uint64_t* dst_offsets;
  EncWs ws;
  int predictor;        // 0 custom Paeth ("L3IF"), 1 original Paeth ("L3IP", reading C16)
};

__device__ __forceinline__ int find_image(const uint64_t* prefix, int n, uint64_t u) {
  int lo = 0, hi = n;
  while (hi - lo > 1) {
    int mid = (lo + hi) >> 1;
    if (prefix[mid] <= u) lo = mid; else hi = mid;
  }
  return lo;
}

struct UnitGeom {
  const uint8_t* plane;
  uint32_t W, x0, y0, w, h;
};

__device__ __forceinline__ UnitGeom unit_geom(const EncParams& p, const EncDesc& d, uint32_t ul) {
  UnitGeom g;
  const uint32_t ch = ul / d.P, pp = ul % d.P;
  g.plane = p.images + d.img_off + (uint64_t)ch * d.W * d.H;
  g.W = d.W;
  g.x0 = (pp % d.gx) * d.N;
  g.y0 = (pp / d.gx) * d.N;
  g.w = min(d.N, d.W - g.x0);
  g.h = min(d.N, d.H - g.y0);
  return g;
}

// Residual of column c in row r (row 0 unfiltered, C5). The encoder sees the
// original pixels, so even the original Paeth (left neighbour) is column-parallel here.
__device__ __forceinline__ int residual(const UnitGeom& g, uint32_t r, uint32_t c, int predictor) {
  const uint8_t* row = g.plane + (uint64_t)(g.y0 + r) * g.W + g.x0;
  const int x = row[c];
  if (r == 0) return x;
  const uint8_t* up = row - g.W;
  if (predictor) return (x - paeth_png_pred(c ? row[c - 1] : 0, up[c], c ? up[c - 1] : 0)) & 0xFF;
  const int t = up[c];
  const int tl = c > 0 ? up[c - 1] : t;
  const int tr = c + 1 < g.w ? up[c + 1] : t;
  return (x - paeth_pred(tl, t, tr)) & 0xFF;
}

// Columns per lane: 4 consecutive columns for wide patches, fewer for narrow ones so that all 32
// lanes stay busy (N = 32: one column per lane).
__device__ __forceinline__ uint32_t enc_cpl(uint32_t w) { return w > 64u ? 4u : (w > 32u ? 2u : 1u); }

// The residuals of cpl (<= 4) consecutive columns c0 .. of row r (byte i = column c0+i; columns past
// the patch width are 0) and how many of them are real.
__device__ __forceinline__ uint32_t residual4(const UnitGeom& g, uint32_t r, uint32_t c0, uint32_t cpl, int predictor,
                                              uint32_t* nvalid) {
  const uint32_t nv = c0 < g.w ? min(cpl, g.w - c0) : 0u;
  uint32_t q = 0;
  for (uint32_t i = 0; i < nv; i++) q |= (uint32_t)residual(g, r, c0 + i, predictor) << (8 * i);
  *nvalid = nv;
  return q;
}

// Row base-delta parameters (readings C2/C6) over the residual words of the row, one
// word (4 columns) per lane and 128-column chunk; warp-collective. Rows >= 1 compare residuals as
// signed bytes (reading C2), row 0 (raw pixels) unsigned.
constexpr int kEncChunks = 2;   // 4 columns x 32 lanes x 2 = 256 >= every N (u8 header field)
__device__ __forceinline__ void row_kb4(const uint32_t* q, const uint32_t* nv, uint32_t r, int* k, int* base) {
  int mn = 1 << 20, mx = -(1 << 20);
#pragma unroll
  for (int m = 0; m < kEncChunks; m++)
    for (uint32_t i = 0; i < nv[m]; i++) {
      int v = (int)((q[m] >> (8 * i)) & 0xFFu);
      if (r > 0 && v >= 128) v -= 256;
      mn = min(mn, v);
      mx = max(mx, v);
    }
  mn = __reduce_min_sync(0xffffffffu, mn);
  mx = __reduce_max_sync(0xffffffffu, mx);
  const int span = mx - mn;
  *k = span > 0 ? 32 - __clz(span) : 1;
  *base = mn & 0xFF;
}

// All residual words of row r for this lane: column chunk m covers columns 32 cpl m + cpl lane ...
__device__ __forceinline__ void row_words(const UnitGeom& g, uint32_t r, int lane, int predictor, uint32_t* q,
                                          uint32_t* nv) {
  const uint32_t cpl = enc_cpl(g.w);
#pragma unroll
  for (int m = 0; m < kEncChunks; m++) q[m] = residual4(g, r, 32u * cpl * m + cpl * lane, cpl, predictor, &nv[m]);
}

__global__ void l3_enc_size_kernel(EncParams p) {
  const int lane = threadIdx.x & 31;
  const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x >> 5);
  for (uint64_t u = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); u < p.total_units; u += warps) {
    const int i = find_image(p.ws.unit_prefix, p.n, u);
    const EncDesc d = p.ws.desc[i];
    const UnitGeom g = unit_geom(p, d, (uint32_t)(u - d.unit0));
    uint64_t bits = 0;
    for (uint32_t r = 0; r < g.h; r++) {
      uint32_t q[kEncChunks], nv[kEncChunks];
      row_words(g, r, lane, p.predictor, q, nv);
      int k, base;
      row_kb4(q, nv, r, &k, &base);
      bits += 12u + (uint64_t)k * g.w;
    }
    if (lane == 0) p.ws.unit_bytes[u] = (uint32_t)((bits + 7) / 8);
  }
}

// One CTA per image: exclusive scan of its units' byte counts.
__global__ void __launch_bounds__(1024) l3_enc_scan_kernel(EncParams p) {
  __shared__ uint64_t warp_tot[32];
  __shared__ uint64_t carry_s;
  const int i = blockIdx.x;
  const EncDesc d = p.ws.desc[i];
  const uint64_t nu = 3ull * d.P;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (threadIdx.x == 0) carry_s = 0;
  __syncthreads();
  for (uint64_t b = 0; b < nu; b += blockDim.x) {
    const uint64_t u = b + threadIdx.x;
    const uint64_t v = u < nu ? p.ws.unit_bytes[d.unit0 + u] : 0;
    uint64_t x = v;
    for (int o = 1; o < 32; o <<= 1) {
      uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[wid] = x;
    __syncthreads();
    if (wid == 0) {
      uint64_t wv = lane < (int)(blockDim.x >> 5) ? warp_tot[lane] : 0, z = wv;
      for (int o = 1; o < 32; o <<= 1) {
        uint64_t y = __shfl_up_sync(0xffffffffu, z, o);
        if (lane >= o) z += y;
      }
      warp_tot[lane] = z - wv;
    }
    __syncthreads();
    const uint64_t excl = carry_s + warp_tot[wid] + x - v;
    if (u < nu) p.ws.unit_off[d.unit0 + u] = (uint32_t)excl;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry_s = excl + v;
    __syncthreads();
  }
  if (threadIdx.x == 0) p.ws.file_size[i] = (uint64_t)d.hdr + carry_s;
}

__global__ void l3_enc_files_kernel(EncParams p) {
  if (threadIdx.x == 0) {
    uint64_t acc = 0;
    for (int i = 0; i < p.n; i++) {
      p.dst_offsets[i] = acc;
      acc += p.ws.file_size[i];
    }
    p.dst_offsets[p.n] = acc;
  }
}

// OR the `nbits` (<= 32) MSB-aligned bits of F into the stream at bit position `pos` (reading C8,
// MSB-first): stream words are big-endian in `words` (bit 31 = first bit), so a field touches at
// most two words — two shared-memory atomics per lane and row instead of one per byte and delta.
__device__ __forceinline__ void put_field(uint32_t* words, uint32_t pos, uint32_t F, uint32_t nbits) {
  if (nbits == 0) return;
  const uint32_t w0 = pos >> 5, sh = pos & 31u;
  atomicOr(&words[w0], F >> sh);
  if (sh + nbits > 32u) atomicOr(&words[w0 + 1], F << (32u - sh));
}

// E4: one warp per unit, rows in order. The unit's bitstream is written straight to the file with
// aligned 32-bit stores: bit b of the stream lives in the aligned word holding byte a + b/8, where a =
// the unit's start address mod 4. Each row's fields are ORed into a small per-warp window of words
// in shared memory (two word atomics per lane); after the row, the completed words go to global
// memory and the partial last word moves to the window's front. Words the unit shares with its
// neighbours (its first and last) are written byte by byte. No patch-sized buffer: 8 warps per block.
constexpr int kEncPackWarps = 8;
constexpr uint32_t kEncWin = 80;   // words: the carried word + one row (12 + 8 x 255 bits = 65 words)

__device__ __forceinline__ void enc_store_word(uint8_t* base, uint32_t w, uint32_t word, uint32_t a, uint32_t nbytes) {
  // stream bytes [a, a + nbytes) of the aligned region at base; word w covers bytes [4w, 4w + 4)
  const uint32_t lo = 4u * w, hi = lo + 4u;
  if (lo >= a && hi <= a + nbytes) {
    *reinterpret_cast<uint32_t*>(base + lo) = bswap32(word);
  } else {
#pragma unroll
    for (uint32_t i = 0; i < 4; i++)
      if (lo + i >= a && lo + i < a + nbytes) base[lo + i] = (uint8_t)(word >> (24 - 8 * i));
  }
}

__global__ void __launch_bounds__(kEncPackWarps * 32) l3_enc_pack_kernel(EncParams p) {
  __shared__ uint32_t win_all[kEncPackWarps][kEncWin];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t* win = win_all[warp];
  const uint64_t warps = (uint64_t)gridDim.x * kEncPackWarps;
  for (uint64_t u = (uint64_t)blockIdx.x * kEncPackWarps + warp; u < p.total_units; u += warps) {
    const int i = find_image(p.ws.unit_prefix, p.n, u);
    const EncDesc d = p.ws.desc[i];
    const uint32_t ul = (uint32_t)(u - d.unit0);
    const UnitGeom g = unit_geom(p, d, ul);
    uint8_t* file = p.dst + p.dst_offsets[i];
    const uint32_t nbytes = p.ws.unit_bytes[u];
    const uint32_t off = p.ws.unit_off[u];
    // container fields (Fig. 5; reading C9)
    if (lane < 4) file[13 + 4ull * ul + lane] = (uint8_t)(off >> (8 * lane));
    if (ul == 0 && lane < 13) {
      uint8_t b;
      if (lane < 4) b = (uint8_t)(p.predictor ? "L3IP" : "L3IF")[lane];
      else if (lane < 8) b = (uint8_t)(d.W >> (8 * (lane - 4)));
      else if (lane < 12) b = (uint8_t)(d.H >> (8 * (lane - 8)));
      else b = (uint8_t)d.N;
      file[lane] = b;
    }
    uint8_t* dst = file + d.hdr + off;
    const uint32_t a = (uint32_t)(reinterpret_cast<uintptr_t>(dst) & 3u);
    uint8_t* base = dst - a;                   // aligned start of the unit's words
    const uint32_t span = min(kEncWin, (31u + 12u + 8u * g.w) / 32u + 2u);   // window words one row can touch
    for (uint32_t x = lane; x < span; x += 32) win[x] = 0;
    __syncwarp();
    uint32_t wbase = 0;                        // stream word index of win[0]
    uint32_t pos = 8u * a;                     // bit position of the current row in the aligned stream
    for (uint32_t r = 0; r < g.h; r++) {
      uint32_t q[kEncChunks], nv[kEncChunks];
      row_words(g, r, lane, p.predictor, q, nv);
      int k, base8;
      row_kb4(q, nv, r, &k, &base8);
      const uint32_t wp = pos - 32u * wbase;   // row position inside the window
      if (lane == 0) put_field(win, wp, (((uint32_t)k << 8) | (uint32_t)base8) << 20, 12);
      // a4 in reverse: the lane's deltas (residual - base) mod 256 as one MSB-first k-bit field each
      const uint32_t cpl = enc_cpl(g.w);
#pragma unroll
      for (int m = 0; m < kEncChunks; m++) {
        uint32_t F = 0;
        for (uint32_t t = 0; t < nv[m]; t++) F = (F << k) | ((((q[m] >> (8 * t)) & 0xFFu) - (uint32_t)base8) & 0xFFu);
        const uint32_t nb = nv[m] * (uint32_t)k;
        if (nb) put_field(win, wp + 12u + (32u * cpl * m + cpl * (uint32_t)lane) * (uint32_t)k, F << (32u - nb), nb);
      }
      pos += 12u + (uint32_t)k * g.w;
      __syncwarp();
      // flush the completed words, carry the partial one to the window front
      const uint32_t done = (pos >> 5) - wbase;   // complete words in the window
      for (uint32_t x = lane; x < done; x += 32) enc_store_word(base, wbase + x, win[x], a, nbytes);
      __syncwarp();
      const uint32_t carry = win[done];
      __syncwarp();
      for (uint32_t x = lane; x < span; x += 32) win[x] = (x == 0) ? carry : 0u;
      wbase += done;
      __syncwarp();
    }
    // the last (partial) word: the stream is padded to whole bytes (nbytes), the rest belongs to the next unit
    if (lane == 0 && 32u * wbase < 8u * (a + nbytes)) enc_store_word(base, wbase, win[0], a, nbytes);
    __syncwarp();
  }
}

// ---------------------------------------------------------------- host side
static uint32_t policy_N(uint32_t W, uint32_t H) {
  const uint64_t A = (uint64_t)W * H;
  return A < 777600ull ? 32u : (A < 2073600ull ? 64u : 128u);
}

struct EncPlan {
  std::vector<EncDesc> desc;
  std::vector<uint64_t> prefix;
  uint64_t units = 0;
  uint64_t max_bytes = 0;
  uint32_t worst_patch = 0;
  bool ok = true;
};

static EncPlan plan_encode(const int32_t* shapes, const int32_t* n_host, int32_t n,
                           const uint64_t* img_offsets) {
  EncPlan pl;
  pl.desc.resize(n);
  pl.prefix.resize(n + 1);
  pl.prefix[0] = 0;
  for (int i = 0; i < n; i++) {
    const int32_t H = shapes[2 * i], W = shapes[2 * i + 1];
    int32_t N = n_host ? n_host[i] : 0;
    if (H <= 0 || W <= 0 || N < 0 || N > 255) { pl.ok = false; return pl; }
    if (N == 0) N = (int32_t)policy_N((uint32_t)W, (uint32_t)H);
    EncDesc& d = pl.desc[i];
    d.W = W; d.H = H; d.N = N;
    d.gx = (W + N - 1) / N;
    const uint64_t P = (uint64_t)d.gx * ((H + N - 1) / N);
    if (3 * P >= (1ull << 29)) { pl.ok = false; return pl; }
    d.P = (uint32_t)P;
    d.hdr = (uint32_t)(13 + 12 * P);
    d.img_off = img_offsets ? img_offsets[i] : 0;
    d.unit0 = pl.prefix[i];
    pl.prefix[i + 1] = pl.prefix[i] + 3 * P;
    const uint32_t wn = (uint32_t)N;
    const uint32_t worst = (wn * (12 + 8 * wn) + 7) / 8;
    if (worst > pl.worst_patch) pl.worst_patch = worst;
    pl.max_bytes += l3_encode_max_bytes((uint32_t)W, (uint32_t)H, N);
  }
  pl.units = pl.prefix[n];
  return pl;
}

uint64_t encode_workspace_size(const int32_t* shapes, const int32_t* n_host, int32_t n) {
  EncPlan pl = plan_encode(shapes, n_host, n, nullptr);
  if (!pl.ok) return 0;
  // descriptors + prefix are uploaded in front of the EncWs sections
  return EncWs::bytes(n, pl.units);
}

l3_status_t encode_batch(const l3_encode_args* a, cudaStream_t s) {
  if (!a || a->n < 0 || (a->n > 0 && (!a->images || !a->shapes_host || !a->img_offsets_host || !a->dst ||
                                       !a->dst_offsets || !a->workspace)))
    return L3_E_INVALID_ARGUMENT;
  if (a->predictor != 0 && a->predictor != 1) return L3_E_INVALID_ARGUMENT;
  if (a->n == 0) return L3_OK;
  EncPlan pl = plan_encode(a->shapes_host, a->n_host, a->n, a->img_offsets_host);
  if (!pl.ok) return L3_E_INVALID_ARGUMENT;
  if (a->workspace_bytes < EncWs::bytes(a->n, pl.units) || a->dst_capacity < pl.max_bytes)
    return L3_E_INVALID_ARGUMENT;
  EncWs ws = EncWs::at(a->workspace, a->n, pl.units);
  if (cudaMemcpyAsync(ws.desc, pl.desc.data(), sizeof(EncDesc) * a->n, cudaMemcpyHostToDevice, s) != cudaSuccess)
    return L3_E_CUDA;
  if (cudaMemcpyAsync(ws.unit_prefix, pl.prefix.data(), 8ull * (a->n + 1), cudaMemcpyHostToDevice, s) !=
      cudaSuccess)
    return L3_E_CUDA;
  if (pl.units == 0) return L3_OK;
  EncParams p;
  p.images = a->images;
  p.n = a->n;
  p.total_units = pl.units;
  p.dst = a->dst;
  p.dst_offsets = a->dst_offsets;
  p.ws = ws;
  p.predictor = a->predictor;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const uint64_t want = (pl.units + 7) / 8;
  const int grid1 = (int)(want < (uint64_t)sms * 16 ? (want ? want : 1) : (uint64_t)sms * 16);
  l3_enc_size_kernel<<<grid1, 256, 0, s>>>(p);
  l3_enc_scan_kernel<<<a->n, 1024, 0, s>>>(p);
  l3_enc_files_kernel<<<1, 32, 0, s>>>(p);
  const uint64_t want4 = (pl.units + kEncPackWarps - 1) / kEncPackWarps;
  const int grid4 = (int)(want4 < (uint64_t)sms * 8 ? want4 : (uint64_t)sms * 8);
  l3_enc_pack_kernel<<<grid4, kEncPackWarps * 32, 0, s>>>(p);
  return cudaGetLastError() == cudaSuccess ? L3_OK : L3_E_CUDA;
}

}  // namespace l3
