/*
 * l3.h — C ABI of the B200-native L3 batch decoder (arXiv 2208.08711).
 *
 * The library (paper_2208_08711_b200/libl3_b200.so) decodes batches of L3 files
 * that are already resident in device memory into planar CHW tensors, entirely
 * in hand-written sm_100a kernels. All functions are `extern "C"`, take plain
 * pointers and sizes, never allocate on the call path, and never synchronise
 * the stream unless stated.
 *
 * Format (§4.3 Fig. 5; readings C8/C9 in DESIGN.md §3):
 *   file  = "L3IF" | W u32le | H u32le | N u8 | offR[P] | offG[P] | offB[P] | data
 *   P     = ceil(W/N) * ceil(H/N); offsets are u32le byte offsets relative to
 *           the start of the data section, strictly increasing over R||G||B,
 *           offR[0] = 0; unit u = ch*P + p owns bytes [off[u], off[u+1]) (the
 *           last unit runs to the end of the file).
 *   patch = rows r = 0..h-1, each `k:4 | base:8 | w deltas of k bits`, MSB-first,
 *           rows bit-contiguous, padded to a byte (Fig. 4).
 *   pixel = row 0: base + delta; rows >= 1: pred(TL, T, TR of row r-1) + base +
 *           delta, all mod 256 (Fig. 3), clamp-to-edge
 *           at the patch's columns 0 and w-1, ties TL, T, TR.
 *
 * Error behaviour:
 *   - Argument / launch problems are returned synchronously (L3_E_INVALID_ARGUMENT,
 *     L3_E_CUDA); nothing is enqueued in that case.
 *   - Data problems are reported asynchronously, per image, in `status[i]`
 *     (and `bad_unit[i]`): header problems take precedence
 *     (L3_E_UNRECOGNIZED_FORMAT, L3_E_CORRUPT_HEADER, bad_unit = -1); otherwise
 *     the first failing unit in canonical order ch*P + p with
 *     L3_E_CORRUPT_STREAM (k = 0 or k > 8) or L3_E_TRUNCATED_STREAM (a row
 *     reads past the unit's byte range) — the result of a sequential decode
 *     (SPEC.md:100, 211, 219, 274-279). Other images still decode; the pixels
 *     of a failed image are unspecified.
 *
 * Ownership: the caller owns every buffer; buffers must stay valid until the
 * stream reaches the call. Concurrent calls need distinct workspaces.
 */
#ifndef L3_H
#define L3_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  L3_OK = 0,
  L3_E_INVALID_ARGUMENT = 1,
  L3_E_UNRECOGNIZED_FORMAT = 2,
  L3_E_CORRUPT_HEADER = 3,
  L3_E_CORRUPT_STREAM = 4,
  L3_E_TRUNCATED_STREAM = 5,
  L3_E_CUDA = 6
} l3_status_t;

typedef enum {
  L3_OUT_U8 = 0,   /* uint8 planar [3, H, W] per image (step a6, u8)                   */
  L3_OUT_F32 = 1   /* float32 [3, H, W] per image, y = fmaf((float)x, scale[c], bias[c]) */
} l3_out_kind_t;

/* Opaque CUDA stream handle (cudaStream_t); NULL = legacy default stream. */
typedef void* l3_stream_t;

/*
 * Arguments of one batch decode ("first reads the
 * header of each image and then splits it into multiple patches").
 *   src          device, 16-byte aligned: the batch's files concatenated.
 *   src_offsets  device, n+1 uint64: file i = src[src_offsets[i] .. src_offsets[i+1]).
 *   shapes       device, n x {H, W} int32: the caller's expected shape of image i;
 *                a header that disagrees is L3_E_CORRUPT_HEADER.
 *   out          device: decoded output (u8 or f32 elements per out_kind).
 *   out_offsets  device, n uint64 ELEMENT offsets of image i's [3,H,W] block (or its
 *                [H,W,3] block with L3_DECODE_LAYOUT_HWC), or NULL: image i starts at
 *                element i*3*H_i*W_i (dense [n,3,H,W] / [n,H,W,3] when every shape is equal).
 *   scale, bias  F32 only: per channel (R, G, B).
 *   status       device, n int32 (l3_status_t), written by the call.
 *   bad_unit     device, n int32 or NULL: first failing unit ch*P + p, else -1.
 *   workspace    device, >= l3_decode_workspace_size(n) bytes, 256-byte aligned,
 *                zero-filled before first use (see l3_decode_batch).
 *   flags        L3_DECODE_HINT_* performance hints and L3_DECODE_LAYOUT_HWC (0 = none).
 *   crops        optional: image i is decoded only inside the window rows [y, y+h) x cols
 *                [x, x+w) (flip != 0: mirrored left-right) into a [3, h, w] block (dense:
 *                element i*3*h*w). Only the patches the window touches are read and decoded
 *                (patches are independently addressable); status then covers
 *                the header and those patches. A window outside the image is
 *                L3_E_INVALID_ARGUMENT in status[i]. With L3_DECODE_LAYOUT_HWC the block
 *                is [h, w, 3].
 */
/* l3_decode_args.flags */
#define L3_DECODE_HINT_WIDE 1u   /* u8 out: most files use 33 <= N <= 128 (e.g. policy N = 128 for
                                    >= FHD images): pick the 8-column-per-lane kernel variant.
                                    A performance hint only; every file decodes correctly either way.
                                    Ignored for L3_OUT_F32 and with crops. */
#define L3_DECODE_LAYOUT_HWC 2u  /* f3: interleaved output, element (y, x, c) of image i
                                    at out_offsets[i] + (y * W + x) * 3 + c (W = window width with
                                    crops), u8 or f32 per out_kind; the channel planes of the file
                                     are interleaved in the store epilogue. */

typedef struct {
  const uint8_t* src;
  const uint64_t* src_offsets;
  const int32_t* shapes;
  int32_t n;
  int32_t out_kind;
  void* out;
  const uint64_t* out_offsets;
  float scale[3];
  float bias[3];
  int32_t* status;
  int32_t* bad_unit;
  void* workspace;
  uint64_t workspace_bytes;
  uint32_t flags;   /* L3_DECODE_HINT_* bits, 0 = none */
  uint32_t max_ctas;      /* 0: the persistent decode grid covers every SM (SMs x resident CTAs);
                             else at most max_ctas thread blocks, i.e. the decoder's share of the
                             GPU is capped so that a concurrent (higher-priority) compute kernel
                             keeps the remaining SMs ("We prioritize the computing
                             stream over the decoding stream"). Any value decodes correctly. */
  const int32_t* crops;   /* device, n x {y, x, h, w, flip} or NULL (partial decode) */
} l3_decode_args;

/* Bytes of device workspace one l3_decode_batch call over n images needs. */
uint64_t l3_decode_workspace_size(int32_t n);

/*
 * The whole hot path, asynchronously on `stream`, as
 * one or two launches (l3_decode_launches): a one-block kernel parses the headers and
 * decomposes the work (a1), and the persistent patch decoder on every SM (staging,
 * row-header chain, delta unpack, row-parallel custom Paeth, store / fused normalise;
 * a2-a6) is launched as its programmatic dependent: its blocks are resident and set
 * up before a1 ends and start decoding as soon as a1's results are visible. Planar
 * batches of up to 32 images (no crop, no HWC) run a1 inside every decoder block
 * instead (one launch). The last decoder block writes the per-image status (a7).
 * The workspace must be zero-filled before its first use (e.g. cudaMemsetAsync);
 * every call leaves it zero-filled again, so it can be reused without host work.
 */
l3_status_t l3_decode_batch(const l3_decode_args* args, l3_stream_t stream);

/* Step a1 alone (header validation, status of header-level errors, work
 * decomposition into the workspace); decodes nothing. */
l3_status_t l3_parse_batch(const l3_decode_args* args, l3_stream_t stream);

/*
 * Load + decode (PAPER.md:67 Load stage, :189 decode on its own stream):
 * copies host_src (pinned host memory, host_src_bytes = src_offsets[n] bytes)
 * into args->src (device) with cudaMemcpyAsync on `stream`, decodes, and
 * copies the n statuses back into host_status (pinned host, n int32). The call
 * is asynchronous; host_status is valid after the stream is synchronised.
 */
l3_status_t l3_load_decode_batch(const l3_decode_args* args, const void* host_src,
                                 uint64_t host_src_bytes, int32_t* host_status,
                                 l3_stream_t stream);

/* The most kernels one l3_decode_batch call launches (2: the a1 kernel and the decode grid). */
int32_t l3_decode_kernels_per_call(void);

/* Kernels the l3_decode_batch call with these arguments launches: 1 when a1 runs inside the decode
 * grid (planar, not crop, not HWC, n <= 32), 2 otherwise, 0 for n == 0; -1 if the
 * arguments are invalid (the same checks as l3_decode_batch). Host-only, no device work. */
int32_t l3_decode_launches(const l3_decode_args* a);

/*
 * Ablation decoders (§5.5 Fig. 10), u8 output, valid files
 * only (statuses cover the header; stream errors are not detected), for timing comparisons:
 *   mode 0  one thread per patch, sequential base-delta + sequential Paeth
 *   mode 1  one warp per patch, pixel-wise parallel base-delta, sequential Paeth
 *   mode 2  one warp per patch, sequential base-delta, row-wise parallel Paeth
 *   mode 3  one warp per patch, both parallel (the paper's design, plain scalar code)
 *   mode 4  one warp per patch, sequential base-delta + sequential Paeth (lane 0)
 *   mode 5  one warp per patch staged in shared memory: pixel-wise base-delta, then an
 *           anti-diagonal wavefront (original Paeth) or row-parallel (custom Paeth) reconstruction
 * Modes 0, 1, 4 and 5 also read the original-Paeth variant "L3IP" (per image, by magic; reading
 * C16), so the paper's Baseline / +Pixel-wise BD bars are modes 0 / 1 on L3IP files. Modes 2
 * and 3 cannot (the left dependency forbids a row-parallel Paeth) and set L3IP images to
 * L3_E_UNRECOGNIZED_FORMAT. Other modes: L3_E_INVALID_ARGUMENT.
 * Same arguments as l3_decode_batch (out_kind must be L3_OUT_U8, crops NULL).
 */
l3_status_t l3_decode_batch_ablation(const l3_decode_args* args, int32_t mode, l3_stream_t stream);

/*
 * Diagnostic: evaluates the decoder's device-side custom-Paeth predictor
 * (Fig. 3; ties TL, T, TR) on all 2^24 triples.
 * out: device, 2^24 bytes; out[TL<<16 | T<<8 | TR] = predicted byte.
 */
l3_status_t l3_selftest_paeth(uint8_t* out, l3_stream_t stream);

/* Exhaustive self-test of the byte-form 4-sample predictor used by the planar
 * and crop decode paths (same rule, Fig. 3; ties TL, T, TR): for
 * every triple and every sample position q in 0..3 of a lane's 4 columns.
 * out: device, 4 * 2^24 bytes; out[q << 24 | TL<<16 | T<<8 | TR] = predicted byte.
 * Returns INVALID_ARGUMENT for a NULL out, CUDA on a launch error; async. */
l3_status_t l3_selftest_paeth4(uint8_t* out, l3_stream_t stream);

/* Exhaustive self-test of the biased-half (fp16x2) predictor used by the fp32
 * planar and crop decode paths (same rule, Fig. 3; ties TL, T, TR;
 * samples held as the fp16 values 1024 + c).
 * out: device, 2^24 bytes; out[TL<<16 | T<<8 | TR] = predicted byte (0xEE if the
 * result lost its bias byte). Returns INVALID_ARGUMENT for a NULL out, CUDA on a
 * launch error; async. */
l3_status_t l3_selftest_paeth_h2(uint8_t* out, l3_stream_t stream);

/* Human-readable name of a status code; never NULL. */
const char* l3_status_string(int32_t status);

/* ------------------------------------------------------------------------ */
/* GPU encoder. Offline dataset          */
/* conversion, byte-identical to the CPU oracle's encoder (reading C2 base).  */
/* ------------------------------------------------------------------------ */

/* PAPER.md:166 patch-size policy (reading C10): pixel count < 777,600 -> 32,
 * < 2,073,600 -> 64, else 128. */
int32_t l3_choose_patch_size(uint32_t W, uint32_t H);

/* Upper bound of the file size of a W x H image with patch size N (0 = policy). */
uint64_t l3_encode_max_bytes(uint32_t W, uint32_t H, int32_t N);

/*
 * Arguments of one batch encode. Shapes and patch sizes are HOST arrays (an
 * offline encoder knows its images); images and outputs live on the device.
 *   images       device: image i is planar uint8 [3, H, W] at images + img_offsets_host[i].
 *   shapes_host  host, n x {H, W}.
 *   n_host       host, n patch sizes (0 = policy) or NULL (policy for all).
 *   dst          device, dst_capacity >= sum of l3_encode_max_bytes.
 *   dst_offsets  device, n+1 uint64, written: file i = dst[dst_offsets[i] .. dst_offsets[i+1]).
 *   predictor    0: the custom Paeth of PAPER.md:137 (magic "L3IF", the hot path's format).
 *                1: the ORIGINAL left/top/top-left Paeth, magic "L3IP": the
 *                   format of the paper's ablation baseline (Fig. 10), readable only by
 *                   l3_decode_batch_ablation modes 0 and 1 (reading C16).
 *                Other values: L3_E_INVALID_ARGUMENT.
 */
typedef struct {
  const uint8_t* images;
  const uint64_t* img_offsets_host;
  const int32_t* shapes_host;
  const int32_t* n_host;
  int32_t n;
  uint8_t* dst;
  uint64_t dst_capacity;
  uint64_t* dst_offsets;
  void* workspace;
  uint64_t workspace_bytes;
  int32_t predictor;
} l3_encode_args;

/* Device workspace bytes for l3_encode_batch (depends on the host shapes). */
uint64_t l3_encode_workspace_size(const int32_t* shapes_host, const int32_t* n_host, int32_t n);

/* Encode the batch asynchronously on `stream` (the descriptor upload is a
 * host-to-device copy on the same stream; the host arrays may be reused when
 * the call returns). */
l3_status_t l3_encode_batch(const l3_encode_args* args, l3_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* L3_H */
