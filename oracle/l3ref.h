/*
 * l3ref.h — CPU ORACLE for the L3 codec (arXiv 2208.08711).
 *
 * TEST INFRASTRUCTURE ONLY. Nothing in the product path (paper_2208_08711_b200/,
 * include/) may include, link or call this. Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs use it.
 *
 * Plain, slow, obviously-correct C written from PAPER.md §4.2–§4.3, with every
 * point where the paper is silent resolved by the readings listed in DESIGN.md §3
 * (C1..C14). It shares no code, header, table or helper with the CUDA path.
 *
 * Status codes are part of the documented interface contract;
 * the numeric values are written out here independently of include/l3.h.
 */
#ifndef L3REF_H
#define L3REF_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  L3REF_OK = 0,
  L3REF_E_INVALID_ARGUMENT = 1,
  L3REF_E_UNRECOGNIZED_FORMAT = 2,
  L3REF_E_CORRUPT_HEADER = 3,
  L3REF_E_CORRUPT_STREAM = 4,
  L3REF_E_TRUNCATED_STREAM = 5
};

/* Residual-row base rule (reading C2). */
enum { L3REF_BASE_SIGNED = 0, L3REF_BASE_UNSIGNED = 1 };

/* PAPER.md:135-137 (§4.2, Fig. 3): custom Paeth predictor over the previous row. */
int l3ref_predict(int tl, int t, int tr);
int l3ref_predict_png(int a, int b, int c);
void l3ref_predict_png_many(const uint8_t* a, const uint8_t* b, const uint8_t* c, uint64_t n, uint8_t* out);
void l3ref_predict_many(const uint8_t* tl, const uint8_t* t, const uint8_t* tr, uint64_t n, uint8_t* out);

/* PAPER.md:166 (§4.3): patch-size policy, reading C10. */
int l3ref_choose_patch_size(uint32_t W, uint32_t H);

/* PAPER.md:150 (§4.2, Fig. 4): base-delta of one row. Writes k, base, deltas[w]. */
void l3ref_bd_encode_row(const uint8_t* res, int w, int first_row, int base_rule,
                         int k_extra, int* k, int* base, uint8_t* deltas);

/* Upper bound on the encoded file size for a W×H image with patch size N. */
uint64_t l3ref_max_file_bytes(uint32_t W, uint32_t H, int N);

/*
 * encode one planar RGB8 image (3 planes of H×W, row-major,
 * R then G then B) into an L3 file. N = 0 selects the policy.
 * Returns the file length, or 0 on invalid arguments / insufficient capacity.
 */
uint64_t l3ref_encode_image(const uint8_t* planar, uint32_t W, uint32_t H, int N,
                            int base_rule, int k_extra, uint8_t* out, uint64_t cap);

/* Ablation variant: predictor 1 = original (left/top/top-left) Paeth, magic "L3IP". */
uint64_t l3ref_encode_image_variant(const uint8_t* planar, uint32_t W, uint32_t H, int N, int predictor,
                                    uint8_t* out, uint64_t cap);
int l3ref_decode_image_variant(const uint8_t* file, uint64_t len, uint8_t* out, uint64_t out_cap,
                               uint32_t* W, uint32_t* H);

/*
 * Sequential decode of one L3 file.
 * exp_W / exp_H: the caller's expected shape (0 = do not check).
 * out: 3×H×W planar bytes (caller-owned, sized from the header or expected shape).
 * Returns a status; *bad_unit = first failing unit ch*P+p, or -1.
 * Header fields are returned through W/H/N/P if non-NULL (valid when status
 * is not UNRECOGNIZED_FORMAT and the first 13 bytes exist).
 */
int l3ref_decode_image(const uint8_t* file, uint64_t len, uint32_t exp_W, uint32_t exp_H,
                       uint8_t* out, uint64_t out_cap, int64_t* bad_unit,
                       uint32_t* W, uint32_t* H, int* N, uint64_t* P);

/*
 * Batch decode: files concatenated in src, file i =
 * src[src_offsets[i] .. src_offsets[i+1]); shapes = n×{H,W}; output of image i
 * at out + out_offsets[i] (bytes), 3×H×W planar. Units of all images are spread
 * over `threads` POSIX threads; results do not depend on the thread count.
 */
void l3ref_decode_batch(const uint8_t* src, const uint64_t* src_offsets, const int32_t* shapes,
                        int n, uint8_t* out, const uint64_t* out_offsets,
                        int32_t* status, int32_t* bad_unit, int threads);

/* fp64 normalisation definition (reading C14): y = (x/255 - mean)/std. */
void l3ref_normalize(const uint8_t* x, uint64_t count_per_channel, int channels,
                     const double* mean, const double* std, double* y);

#ifdef __cplusplus
}
#endif
#endif
