// l3_ablation.cu — the paper's decoder ablation (§5.5, Fig. 10 `fig:module`)
// re-run on B200, on the same L3 format as the hot path.
//
// The paper's axes, all with patch-level parallelism (its "baseline" state):
//   mode 0  one THREAD per patch: sequential base-delta decode + sequential Paeth
//   mode 1  one WARP per patch: pixel-wise parallel BD, sequential Paeth (lane 0)
//   mode 2  one WARP per patch: sequential BD (lane 0), row-wise parallel Paeth
//   mode 3  one WARP per patch: both (the paper's full design, plain scalar code)
//   mode 4  one WARP per patch: sequential BD + sequential Paeth (lane 0): modes 4 -> 1 isolate
//           the pixel-wise BD step from the thread-vs-warp mapping that modes 0 -> 1 also change
//   mode 5  one WARP per patch in shared memory: pixel-wise BD, then an anti-diagonal wavefront
//           for the original Paeth or row-parallel for the custom Paeth
// The paper's baseline uses the ORIGINAL (left/top/top-left) Paeth. Its format variant "L3IP"
// (reading C16) is decoded by modes 0, 1, 4 (sequential Paeth) and 5 (wavefront); modes 2 and 3
// (row-parallel Paeth) need the custom-Paeth format and report L3IP images as
// UNRECOGNIZED_FORMAT. The paper's four bars are: mode 0 on L3IP (Baseline), mode 1 on L3IP
// (+Pixel-wise BD), mode 2 on L3IF (+Custom Paeth), mode 3 on L3IF (both). The production
// kernel (l3_decode_batch) is the fifth bar.
// Valid files only (the ablation reports time, not errors); reads stay inside each unit.
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/l3.h"
#include "l3_internal.cuh"

namespace l3 {

cudaError_t launch_parse(const l3_decode_args* a, cudaStream_t s, bool accept_variant);

struct AblParams {
  const uint8_t* src;
  uint8_t* out;
  const ImgDesc* desc;
  const int32_t* status;
  int n;
};

__device__ __forceinline__ uint32_t abl_u32le(const uint8_t* p) {
  return (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) | ((uint32_t)p[3] << 24);
}

// k (<= 8) bits at bit position pos of [data, data+len) MSB-first; 0 past the end. A 16-bit
// window of the two bytes holding the field (pos & 7 + k <= 15), as plain scalar code would.
__device__ __forceinline__ uint32_t abl_bits(const uint8_t* data, uint64_t len, uint64_t pos, uint32_t k) {
  const uint64_t b = pos >> 3;
  const uint32_t hi = b < len ? data[b] : 0u, lo = b + 1 < len ? data[b + 1] : 0u;
  const uint32_t win = (hi << 8) | lo;
  return (win >> (16u - (uint32_t)(pos & 7) - k)) & ((1u << k) - 1u);
}

struct AblUnit {
  const uint8_t* data;
  uint64_t len;
  uint8_t* plane;
  uint32_t W, x0, y0, w, h;
  bool png;   // original-Paeth variant (L3IP)
};

__device__ __forceinline__ bool abl_unit(const AblParams& p, int img, uint32_t u, AblUnit& U) {
  const ImgDesc& d = p.desc[img];
  const uint32_t nunits = 3u * d.P;
  if (u >= nunits) return false;
  const uint8_t* file = p.src + d.file_off;
  const uint64_t off = abl_u32le(file + 13 + 4ull * u);
  const uint64_t nxt = (u + 1 < nunits) ? (uint64_t)abl_u32le(file + 17 + 4ull * u) : d.data_len;
  if (unit_offsets_bad(u, nunits, off, nxt, d.data_len)) return false;
  const uint32_t ch = u / d.P, pp = u % d.P;
  U.data = p.src + d.data_off + off;
  U.len = nxt - off;
  U.W = d.W;
  U.x0 = (pp % d.gx) * d.N;
  U.y0 = (pp / d.gx) * d.N;
  U.w = min(d.N, d.W - U.x0);
  U.h = min(d.N, d.H - U.y0);
  U.plane = p.out + d.out_off + (uint64_t)ch * d.W * d.H;
  U.png = is_png_variant(file);
  return true;
}

__device__ __forceinline__ uint64_t abl_image_units(const AblParams& p, int img) {
  return p.status[img] == L3_OK ? 3ull * p.desc[img].P : 0ull;
}

// Walks the batch's units in one flat index space (every unit of every image is available to
// every worker at once); g only grows per worker, so the image cursor advances monotonically.
struct AblCursor {
  int img = 0;
  uint64_t base = 0;
  __device__ __forceinline__ bool seek(const AblParams& p, uint64_t g, uint32_t& u) {
    while (img < p.n) {
      const uint64_t nu = abl_image_units(p, img);
      if (g < base + nu) break;
      base += nu;
      img++;
    }
    if (img >= p.n) return false;
    u = (uint32_t)(g - base);
    return true;
  }
};

// Sequential decode of one unit by one thread, straight into the output plane (modes 0, 5 fallback).
__device__ void abl_seq_unit(const AblUnit& U) {
  uint64_t pos = 0;
  for (uint32_t r = 0; r < U.h; r++) {
    const uint32_t k = min(abl_bits(U.data, U.len, pos, 4), 8u), base = abl_bits(U.data, U.len, pos + 4, 8);
    pos += 12;
    uint8_t* row = U.plane + (uint64_t)(U.y0 + r) * U.W + U.x0;
    for (uint32_t c = 0; c < U.w; c++, pos += k) {
      const int res = (int)((base + abl_bits(U.data, U.len, pos, k)) & 0xFFu);
      if (r == 0) {
        row[c] = (uint8_t)res;
      } else if (U.png) {   // left neighbour = the pixel just decoded (row-wise dependency)
        const uint8_t* up = row - U.W;
        const int a = c ? row[c - 1] : 0, cc = c ? up[c - 1] : 0;
        row[c] = (uint8_t)((paeth_png_pred(a, up[c], cc) + res) & 0xFF);
      } else {
        const uint8_t* up = row - U.W;
        const int t = up[c], tl = c ? up[c - 1] : t, tr = (c + 1 < U.w) ? up[c + 1] : t;
        row[c] = (uint8_t)((paeth_pred(tl, t, tr) + res) & 0xFF);
      }
    }
  }
}

// mode 0: one thread per patch, everything sequential
__global__ void l3_ablation_thread_kernel(AblParams p) {
  const uint64_t tid = blockIdx.x * blockDim.x + threadIdx.x, nth = gridDim.x * blockDim.x;
  AblCursor cur;
  uint32_t u;
  for (uint64_t g = tid; cur.seek(p, g, u); g += nth) {
    AblUnit U;
    if (abl_unit(p, cur.img, u, U)) abl_seq_unit(U);
  }
}

// mode 5: one warp per patch, staged in shared memory: row-header chain (lane 0), pixel-wise BD
// over the whole patch, then the most parallel Paeth order each format allows: an anti-diagonal
// WAVEFRONT for the original Paeth (pixel (r, c) needs (r, c-1), (r-1, c), (r-1, c-1), all on
// earlier diagonals r + c; h + w - 2 dependent steps) and row-parallel for the custom Paeth (h - 1
// steps). Patches above 128 x 128 fall back to lane 0 sequential (N > 128 is outside the policy).
constexpr uint32_t kWaveCap = 16384, kWaveRows = 128, kWaveWarps = 4;
constexpr uint32_t kWaveSmem = kWaveWarps * (kWaveCap + kWaveRows * 6);

__global__ void __launch_bounds__(kWaveWarps * 32) l3_ablation_wave_kernel(AblParams p) {
  extern __shared__ __align__(16) uint8_t wsm[];
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  uint8_t* px = wsm + wl * kWaveCap;
  uint32_t* hpos = reinterpret_cast<uint32_t*>(wsm + kWaveWarps * kWaveCap) + wl * kWaveRows;
  uint8_t* hk = wsm + kWaveWarps * (kWaveCap + 4 * kWaveRows) + wl * kWaveRows;
  uint8_t* hb = hk + kWaveWarps * kWaveRows;
  const uint64_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  AblCursor cur;
  uint32_t u;
  for (uint64_t g = gw; cur.seek(p, g, u); g += nw) {
    AblUnit U;
    if (!abl_unit(p, cur.img, u, U)) continue;
    const uint32_t w = U.w, h = U.h;
    if (h > kWaveRows || w * h > kWaveCap) {
      if (lane == 0) abl_seq_unit(U);
      __syncwarp();
      continue;
    }
    if (lane == 0) {   // a3: the row-header chain is serial by construction
      uint64_t pos = 0;
      for (uint32_t r = 0; r < h; r++) {
        const uint32_t k = min(abl_bits(U.data, U.len, pos, 4), 8u);
        hk[r] = (uint8_t)k;
        hb[r] = (uint8_t)abl_bits(U.data, U.len, pos + 4, 8);
        hpos[r] = (uint32_t)(pos + 12);
        pos += 12 + (uint64_t)k * w;
      }
    }
    __syncwarp();
    for (uint32_t i = lane; i < w * h; i += 32) {   // a4 for every pixel of the patch
      const uint32_t r = i / w, c = i - r * w, k = hk[r];
      px[i] = (uint8_t)((hb[r] + abl_bits(U.data, U.len, (uint64_t)hpos[r] + (uint64_t)c * k, k)) & 0xFFu);
    }
    __syncwarp();
    if (U.png) {
      for (uint32_t d = 1; d + 1 < h + w; d++) {
        const uint32_t r0 = d + 1 > w ? d + 1 - w : 1u, r1 = min(d, h - 1);
        for (uint32_t r = max(r0, 1u) + lane; r <= r1; r += 32) {
          const uint32_t c = d - r, i = r * w + c;
          const int a = c ? px[i - 1] : 0, b = px[i - w], cc = c ? px[i - w - 1] : 0;
          px[i] = (uint8_t)((paeth_png_pred(a, b, cc) + px[i]) & 0xFF);
        }
        __syncwarp();
      }
    } else {
      for (uint32_t r = 1; r < h; r++) {
        for (uint32_t c = lane; c < w; c += 32) {
          const uint32_t i = r * w + c;
          const int t = px[i - w], tl = c ? px[i - w - 1] : t, tr = (c + 1 < w) ? px[i - w + 1] : t;
          px[i] = (uint8_t)((paeth_pred(tl, t, tr) + px[i]) & 0xFF);
        }
        __syncwarp();
      }
    }
    for (uint32_t i = lane; i < w * h; i += 32) {
      const uint32_t r = i / w, c = i - r * w;
      U.plane[(uint64_t)(U.y0 + r) * U.W + U.x0 + c] = px[i];
    }
    __syncwarp();
  }
}

// modes 1-3: one warp per patch; residuals of the current row pass through shared memory
template <bool PAR_BD, bool PAR_PAETH>
__global__ void l3_ablation_warp_kernel(AblParams p) {
  __shared__ uint8_t res_s[8][256];
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const uint64_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  uint8_t* res = res_s[wl];
  AblCursor cur;
  uint32_t u;
  for (uint64_t g = gw; cur.seek(p, g, u); g += nw) {
    const int img = cur.img;
    {
      AblUnit U;
      if (!abl_unit(p, img, u, U)) continue;
      uint64_t pos = 0;
      for (uint32_t r = 0; r < U.h; r++) {
        const uint32_t k = min(abl_bits(U.data, U.len, pos, 4), 8u), base = abl_bits(U.data, U.len, pos + 4, 8);
        pos += 12;
        // step 2 of PAPER.md:152: deltas + base
        if (PAR_BD) {
          for (uint32_t c = lane; c < U.w; c += 32)
            res[c] = (uint8_t)((base + abl_bits(U.data, U.len, pos + (uint64_t)c * k, k)) & 0xFFu);
        } else if (lane == 0) {
          for (uint32_t c = 0; c < U.w; c++)
            res[c] = (uint8_t)((base + abl_bits(U.data, U.len, pos + (uint64_t)c * k, k)) & 0xFFu);
        }
        __syncwarp();
        pos += (uint64_t)k * U.w;
        uint8_t* row = U.plane + (uint64_t)(U.y0 + r) * U.W + U.x0;
        const uint8_t* up = row - U.W;
        if (PAR_PAETH) {
          for (uint32_t c = lane; c < U.w; c += 32) {
            if (r == 0) {
              row[c] = res[c];
            } else {
              const int t = up[c], tl = c ? up[c - 1] : t, tr = (c + 1 < U.w) ? up[c + 1] : t;
              row[c] = (uint8_t)((paeth_pred(tl, t, tr) + res[c]) & 0xFF);
            }
          }
        } else if (lane == 0) {
          for (uint32_t c = 0; c < U.w; c++) {
            if (r == 0) {
              row[c] = res[c];
            } else if (U.png) {
              const int a = c ? row[c - 1] : 0, cc = c ? up[c - 1] : 0;
              row[c] = (uint8_t)((paeth_png_pred(a, up[c], cc) + res[c]) & 0xFF);
            } else {
              const int t = up[c], tl = c ? up[c - 1] : t, tr = (c + 1 < U.w) ? up[c + 1] : t;
              row[c] = (uint8_t)((paeth_pred(tl, t, tr) + res[c]) & 0xFF);
            }
          }
        }
        __syncwarp();
        __threadfence_block();   // row r visible to all lanes before row r+1 reads it
      }
    }
  }
}

cudaError_t launch_ablation(const l3_decode_args* a, int mode, cudaStream_t s) {
  cudaError_t e = launch_parse(a, s, /*accept_variant=*/mode <= 1 || mode >= 4);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  AblParams p;
  p.src = a->src;
  p.out = reinterpret_cast<uint8_t*>(a->out);
  const WsView ws = WsView::at(a->workspace, a->n);
  p.desc = ws.desc;
  p.status = a->status;
  p.n = a->n;
  if (mode == 0) l3_ablation_thread_kernel<<<sms * 8, 128, 0, s>>>(p);
  else if (mode == 1) l3_ablation_warp_kernel<true, false><<<sms * 8, 256, 0, s>>>(p);
  else if (mode == 2) l3_ablation_warp_kernel<false, true><<<sms * 8, 256, 0, s>>>(p);
  else if (mode == 4) l3_ablation_warp_kernel<false, false><<<sms * 8, 256, 0, s>>>(p);
  else if (mode == 5) {
    e = cudaFuncSetAttribute(l3_ablation_wave_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kWaveSmem);
    if (e != cudaSuccess) return e;
    l3_ablation_wave_kernel<<<sms * 3, kWaveWarps * 32, kWaveSmem, s>>>(p);
  }
  else if (mode == 3) l3_ablation_warp_kernel<true, true><<<sms * 8, 256, 0, s>>>(p);
  return cudaGetLastError();
}

}  // namespace l3
