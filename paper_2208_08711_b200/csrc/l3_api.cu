// l3_api.cu — the C ABI declared in include/l3.h (argument checks + launches).
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/l3.h"
#include "l3_internal.cuh"

namespace l3 {
cudaError_t launch_parse(const l3_decode_args* a, cudaStream_t s, bool accept_variant = false);
cudaError_t launch_decode_batch(const l3_decode_args* a, cudaStream_t s);
bool a1_in_cta_call(const l3_decode_args* a);
cudaError_t launch_selftest_paeth(uint8_t* out, cudaStream_t s);
cudaError_t launch_selftest_paeth4(uint8_t* out, cudaStream_t s);
cudaError_t launch_selftest_paeth_h2(uint8_t* out, cudaStream_t s);
cudaError_t launch_ablation(const l3_decode_args* a, int mode, cudaStream_t s);
uint64_t encode_workspace_size(const int32_t* shapes, const int32_t* n_host, int32_t n);
l3_status_t encode_batch(const l3_encode_args* a, cudaStream_t s);
}  // namespace l3

static l3_status_t check_decode_args(const l3_decode_args* a) {
  if (!a || a->n < 0) return L3_E_INVALID_ARGUMENT;
  if (a->n == 0) return L3_OK;
  if (!a->src || !a->src_offsets || !a->shapes || !a->out || !a->status || !a->workspace)
    return L3_E_INVALID_ARGUMENT;
  if ((reinterpret_cast<uintptr_t>(a->src) & 15) != 0) return L3_E_INVALID_ARGUMENT;
  if ((reinterpret_cast<uintptr_t>(a->workspace) & 255) != 0) return L3_E_INVALID_ARGUMENT;
  if (a->workspace_bytes < l3::WsView::bytes(a->n)) return L3_E_INVALID_ARGUMENT;
  if (a->out_kind != L3_OUT_U8 && a->out_kind != L3_OUT_F32) return L3_E_INVALID_ARGUMENT;
  return L3_OK;
}

extern "C" {

uint64_t l3_decode_workspace_size(int32_t n) { return n < 0 ? 0 : l3::WsView::bytes(n); }

int32_t l3_decode_kernels_per_call(void) { return 2; }

int32_t l3_decode_launches(const l3_decode_args* a) {
  if (check_decode_args(a) != L3_OK) return -1;
  if (a->n == 0) return 0;
  return l3::a1_in_cta_call(a) ? 1 : 2;
}

l3_status_t l3_parse_batch(const l3_decode_args* a, l3_stream_t stream) {
  l3_status_t st = check_decode_args(a);
  if (st != L3_OK || a->n == 0) return st;
  return l3::launch_parse(a, (cudaStream_t)stream) == cudaSuccess ? L3_OK : L3_E_CUDA;
}

l3_status_t l3_decode_batch(const l3_decode_args* a, l3_stream_t stream) {
  l3_status_t st = check_decode_args(a);
  if (st != L3_OK || a->n == 0) return st;
  return l3::launch_decode_batch(a, (cudaStream_t)stream) == cudaSuccess ? L3_OK : L3_E_CUDA;
}

l3_status_t l3_load_decode_batch(const l3_decode_args* a, const void* host_src, uint64_t host_src_bytes,
                                 int32_t* host_status, l3_stream_t stream) {
  l3_status_t st = check_decode_args(a);
  if (st != L3_OK) return st;
  if (a->n == 0) return L3_OK;
  if (!host_src || !host_status) return L3_E_INVALID_ARGUMENT;
  cudaStream_t s = (cudaStream_t)stream;
  if (cudaMemcpyAsync((void*)a->src, host_src, host_src_bytes, cudaMemcpyHostToDevice, s) != cudaSuccess)
    return L3_E_CUDA;
  st = l3_decode_batch(a, stream);
  if (st != L3_OK) return st;
  if (cudaMemcpyAsync(host_status, a->status, sizeof(int32_t) * (size_t)a->n, cudaMemcpyDeviceToHost, s) !=
      cudaSuccess)
    return L3_E_CUDA;
  return L3_OK;
}

l3_status_t l3_decode_batch_ablation(const l3_decode_args* a, int32_t mode, l3_stream_t stream) {
  l3_status_t st = check_decode_args(a);
  if (st != L3_OK || a->n == 0) return st;
  if (mode < 0 || mode > 5 || a->out_kind != L3_OUT_U8 || a->crops) return L3_E_INVALID_ARGUMENT;
  return l3::launch_ablation(a, mode, (cudaStream_t)stream) == cudaSuccess ? L3_OK : L3_E_CUDA;
}

l3_status_t l3_selftest_paeth(uint8_t* out, l3_stream_t stream) {
  if (!out) return L3_E_INVALID_ARGUMENT;
  return l3::launch_selftest_paeth(out, (cudaStream_t)stream) == cudaSuccess ? L3_OK : L3_E_CUDA;
}

l3_status_t l3_selftest_paeth4(uint8_t* out, l3_stream_t stream) {
  if (!out) return L3_E_INVALID_ARGUMENT;
  return l3::launch_selftest_paeth4(out, (cudaStream_t)stream) == cudaSuccess ? L3_OK : L3_E_CUDA;
}

l3_status_t l3_selftest_paeth_h2(uint8_t* out, l3_stream_t stream) {
  if (!out) return L3_E_INVALID_ARGUMENT;
  return l3::launch_selftest_paeth_h2(out, (cudaStream_t)stream) == cudaSuccess ? L3_OK : L3_E_CUDA;
}

const char* l3_status_string(int32_t s) {
  switch (s) {
    case L3_OK: return "ok";
    case L3_E_INVALID_ARGUMENT: return "invalid argument";
    case L3_E_UNRECOGNIZED_FORMAT: return "unrecognized format";
    case L3_E_CORRUPT_HEADER: return "corrupt header";
    case L3_E_CORRUPT_STREAM: return "corrupt stream";
    case L3_E_TRUNCATED_STREAM: return "truncated stream";
    case L3_E_CUDA: return "cuda error";
    default: return "unknown status";
  }
}

int32_t l3_choose_patch_size(uint32_t W, uint32_t H) {
  const uint64_t A = (uint64_t)W * H;
  return A < 777600ull ? 32 : (A < 2073600ull ? 64 : 128);
}

uint64_t l3_encode_max_bytes(uint32_t W, uint32_t H, int32_t N) {
  if (W == 0 || H == 0 || N < 0 || N > 255) return 0;
  if (N == 0) N = l3_choose_patch_size(W, H);
  const uint64_t gx = (W + (uint64_t)N - 1) / N, gy = (H + (uint64_t)N - 1) / N, P = gx * gy;
  // per channel: every row at most 12 + 8w bits, each patch padded by < 1 byte
  const uint64_t per_ch = (12ull * H * gx + 8ull * (uint64_t)W * H) / 8ull + 2 * P;
  return 13ull + 12ull * P + 3ull * per_ch;
}

uint64_t l3_encode_workspace_size(const int32_t* shapes_host, const int32_t* n_host, int32_t n) {
  if (n < 0 || (n > 0 && !shapes_host)) return 0;
  return l3::encode_workspace_size(shapes_host, n_host, n);
}

l3_status_t l3_encode_batch(const l3_encode_args* a, l3_stream_t stream) {
  return l3::encode_batch(a, (cudaStream_t)stream);
}

}  // extern "C"
