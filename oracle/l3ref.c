/*
 * l3ref.c — CPU ORACLE for the L3 codec (arXiv 2208.08711).
 *
 * TEST INFRASTRUCTURE ONLY (see l3ref.h). This file is deliberately plain and
 * slow: one pixel at a time, one bit at a time, in the order the paper describes
 * the algorithm. Build: gcc -O2 -std=c11 -fPIC -shared -pthread (no fast-math).
 *
 * Citations are PAPER.md line numbers with section / figure:
 *   §4.2 custom Paeth filter ......... PAPER.md:135-139 (Fig. 3 `fig:paeth`)
 *   §4.2 base-delta encode/decode .... PAPER.md:150-152 (Fig. 4 `fig:bd`)
 *   §4.3 patches, policy, file format  PAPER.md:166-168 (Fig. 5 `fig:file`)
 * Readings C1..C14 (where the paper is silent) are listed in DESIGN.md §3.
 *
 * Parity pins: tests/test_oracle_*.py (Fig. 3 numbers, SPEC vectors, Table 4
 * Black/Random closed forms, exhaustive predictor reformulation, brute-force
 * pure-Python model on tiny inputs, losslessness).
 */
#include "l3ref.h"

#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* §4.2 Custom Paeth predictor                            */
/* ------------------------------------------------------------------------ */

static int iabs_(int x) { return x < 0 ? -x : x; }

/*
 * "the Paeth filter calculates the reference value using those three
 * neighboring pixels as follows: Top_Left + Top_Right - Top (Step 1). Then,
 * among the three neighboring pixels, the filter selects the one whose value
 * is the closest to the reference value (Step 2)."
 * Reading C3: ties resolved in the order TL, T, TR (first minimum wins).
 * The reference value is computed over the integers (no clamping).
 */
int l3ref_predict(int tl, int t, int tr) {
  int ref = tl + tr - t;                /* Step 1 */
  int cand[3] = {tl, t, tr};            /* candidate order = tie order (C3) */
  int best = 0;
  for (int i = 1; i < 3; i++)           /* Step 2: closest candidate */
    if (iabs_(cand[i] - ref) < iabs_(cand[best] - ref)) best = i;
  return cand[best];
}

/*
 * The ORIGINAL Paeth predictor ("the original Paeth filter encodes each
 * pixel based on three neighboring pixels (left, top, top-left)"), as defined for PNG:
 * p = a + b - c; the neighbour closest to p, ties in the order a (left), b (top),
 * c (top-left). Used only by the ablation format variant "L3IP" (reading
 * C16 in DESIGN.md: missing left / top-left neighbours at column 0 are 0, as in PNG).
 */
int l3ref_predict_png(int a, int b, int c) {
  int p = a + b - c;
  int pa = iabs_(p - a), pb = iabs_(p - b), pc = iabs_(p - c);
  if (pa <= pb && pa <= pc) return a;
  if (pb <= pc) return b;
  return c;
}

/* Element-wise l3ref_predict over arrays (lets tests sweep all 2^24 triples). */
void l3ref_predict_many(const uint8_t* tl, const uint8_t* t, const uint8_t* tr, uint64_t n, uint8_t* out) {
  for (uint64_t i = 0; i < n; i++) out[i] = (uint8_t)l3ref_predict(tl[i], t[i], tr[i]);
}

/* Element-wise l3ref_predict_png (a = left, b = top, c = top-left). */
void l3ref_predict_png_many(const uint8_t* a, const uint8_t* b, const uint8_t* c, uint64_t n, uint8_t* out) {
  for (uint64_t i = 0; i < n; i++) out[i] = (uint8_t)l3ref_predict_png(a[i], b[i], c[i]);
}

/* ------------------------------------------------------------------------ */
/* §4.3 Patch-size policy, reading C10                          */
/* ------------------------------------------------------------------------ */

/* "N=32 for images whose resolution is below 1080x720 (HD), N=64 ... between
 * 1080x720 (HD) and 1920x1080 (FHD), and N=128 ... between 1920x1080 (FHD)
 * and 3840x2160 (UHD)" — by pixel count, boundaries assigned upward (C10). */
int l3ref_choose_patch_size(uint32_t W, uint32_t H) {
  uint64_t A = (uint64_t)W * (uint64_t)H;
  if (A < 1080ull * 720ull) return 32;
  if (A < 1920ull * 1080ull) return 64;
  return 128;
}

/* ------------------------------------------------------------------------ */
/* MSB-first bit cursor (reading C8)                                         */
/* ------------------------------------------------------------------------ */

typedef struct {
  uint8_t* buf;
  uint64_t cap_bits;
  uint64_t pos; /* bit position */
  int overflow;
} bitwriter;

static void bw_put(bitwriter* w, uint32_t value, int nbits) {
  for (int i = nbits - 1; i >= 0; i--) {           /* most significant bit first */
    if (w->pos >= w->cap_bits) { w->overflow = 1; return; }
    uint32_t bit = (value >> i) & 1u;
    if (bit) w->buf[w->pos >> 3] |= (uint8_t)(0x80u >> (w->pos & 7));
    w->pos++;
  }
}

typedef struct {
  const uint8_t* buf;
  uint64_t len_bits;
  uint64_t pos;
} bitreader;

/* Returns 0 when fewer than nbits remain (-> TRUNCATED_STREAM). */
static int br_get(bitreader* r, int nbits, uint32_t* value) {
  if (r->len_bits - r->pos < (uint64_t)nbits || r->pos > r->len_bits) return 0;
  uint32_t v = 0;
  for (int i = 0; i < nbits; i++) {
    uint32_t bit = (r->buf[r->pos >> 3] >> (7 - (r->pos & 7))) & 1u;
    v = (v << 1) | bit;
    r->pos++;
  }
  *value = v;
  return 1;
}

/* ------------------------------------------------------------------------ */
/* §4.2 Base-delta encoding of one row                         */
/* ------------------------------------------------------------------------ */

static int bitlen_(int v) { int n = 0; while (v > 0) { n++; v >>= 1; } return n; }

/*
 * "First, each row's minimum and maximum values are found (Step 1). The
 * minimum value is selected as the base value of each row. Also, the minimum
 * number of bits required to cover all delta values is computed (Step 2).
 * Then, the deltas from the base value for all elements are calculated
 * (Step 3)."
 * Reading C2: rows >= 1 hold Paeth residuals, which are differences; they are
 * compared as signed int8 (two's complement of the stored byte). The first
 * (unfiltered, raw pixel) row is compared unsigned. BASE_UNSIGNED selects the
 * alternative reading (unsigned for every row); the decoder is the same.
 * Reading C6: k = max(1, bits(max-min)). k_extra > 0 writes a non-minimal k
 * (valid per reading C7; used only to test decoder generality).
 */
void l3ref_bd_encode_row(const uint8_t* res, int w, int first_row, int base_rule,
                         int k_extra, int* k, int* base, uint8_t* deltas) {
  int is_signed = (!first_row && base_rule == L3REF_BASE_SIGNED);
  int mn = 0, mx = 0;
  for (int c = 0; c < w; c++) {                    /* Step 1: min and max */
    int v = res[c];
    if (is_signed && v >= 128) v -= 256;
    if (c == 0 || v < mn) mn = v;
    if (c == 0 || v > mx) mx = v;
  }
  int kk = bitlen_(mx - mn);                       /* Step 2: bits for the span */
  if (kk < 1) kk = 1;
  kk += k_extra;
  if (kk > 8) kk = 8;
  *k = kk;
  *base = mn & 0xFF;                               /* the minimum is the base */
  for (int c = 0; c < w; c++)                      /* Step 3: deltas */
    deltas[c] = (uint8_t)((res[c] - *base) & 0xFF);
}

/* ------------------------------------------------------------------------ */
/* §4.3 Geometry, reading C9                                  */
/* ------------------------------------------------------------------------ */

static uint64_t ceil_div_(uint64_t a, uint64_t b) { return (a + b - 1) / b; }

uint64_t l3ref_max_file_bytes(uint32_t W, uint32_t H, int N) {
  if (N <= 0) N = l3ref_choose_patch_size(W, H);
  uint64_t gx = ceil_div_(W, (uint64_t)N), gy = ceil_div_(H, (uint64_t)N);
  uint64_t P = gx * gy;
  /* every row at most 12 + 8w bits; each patch padded by < 1 byte */
  uint64_t data = 3ull * ((12ull * H * gx + 8ull * (uint64_t)W * H + 7ull * P) / 8ull + P + 1);
  return 13ull + 12ull * P + data;
}

static void put_u32le_(uint8_t* p, uint32_t v) {
  p[0] = (uint8_t)v; p[1] = (uint8_t)(v >> 8); p[2] = (uint8_t)(v >> 16); p[3] = (uint8_t)(v >> 24);
}
static uint32_t get_u32le_(const uint8_t* p) {
  return (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) | ((uint32_t)p[3] << 24);
}

/* ------------------------------------------------------------------------ */
/* Encoder: §4.2 two stages per patch, §4.3 container     */
/* ------------------------------------------------------------------------ */

static uint64_t encode_image_(const uint8_t* planar, uint32_t W, uint32_t H, int N, int base_rule, int k_extra,
                              int predictor, uint8_t* out, uint64_t cap);

uint64_t l3ref_encode_image(const uint8_t* planar, uint32_t W, uint32_t H, int N,
                            int base_rule, int k_extra, uint8_t* out, uint64_t cap) {
  return encode_image_(planar, W, H, N, base_rule, k_extra, 0, out, cap);
}

/* Ablation variant (f2): predictor 1 = original Paeth, file magic "L3IP". */
uint64_t l3ref_encode_image_variant(const uint8_t* planar, uint32_t W, uint32_t H, int N, int predictor,
                                    uint8_t* out, uint64_t cap) {
  return encode_image_(planar, W, H, N, L3REF_BASE_SIGNED, 0, predictor, out, cap);
}

static uint64_t encode_image_(const uint8_t* planar, uint32_t W, uint32_t H, int N, int base_rule, int k_extra,
                              int predictor, uint8_t* out, uint64_t cap) {
  if (W == 0 || H == 0 || N < 0 || N > 255) return 0;
  if (N == 0) N = l3ref_choose_patch_size(W, H);
  uint64_t gx = ceil_div_(W, (uint64_t)N), gy = ceil_div_(H, (uint64_t)N);
  uint64_t P = gx * gy;
  uint64_t hdr = 13ull + 12ull * P;
  if (cap < hdr) return 0;
  memset(out, 0, (size_t)cap);
  /* Fig. 5: magic (4 B), width (4 B), height (4 B), patch size (1 B), 3 offset arrays */
  memcpy(out, predictor ? "L3IP" : "L3IF", 4);
  put_u32le_(out + 4, W);
  put_u32le_(out + 8, H);
  out[12] = (uint8_t)N;

  bitwriter bw = {out + hdr, (cap - hdr) * 8ull, 0, 0};
  uint8_t* patch = (uint8_t*)malloc((size_t)N * N);
  uint8_t* resid = (uint8_t*)malloc((size_t)N * N);
  uint8_t* deltas = (uint8_t*)malloc((size_t)N);

  /* "the image is first separated into three channels (R, G, and B). Then, the
   * image is divided into square-sized patches for each channel, and the
   * encoding algorithm is applied to each patch." */
  for (int ch = 0; ch < 3; ch++) {
    const uint8_t* plane = planar + (uint64_t)ch * W * H;
    for (uint64_t p = 0; p < P; p++) {
      uint64_t px = p % gx, py = p / gx;                  /* row-major patch order */
      int x0 = (int)(px * N), y0 = (int)(py * N);
      int w = (int)((W - x0) < (uint32_t)N ? (W - x0) : (uint32_t)N);
      int h = (int)((H - y0) < (uint32_t)N ? (H - y0) : (uint32_t)N);
      /* "the offset for each patch is recorded" — byte offset from data start (C9) */
      put_u32le_(out + 13 + 4ull * ((uint64_t)ch * P + p), (uint32_t)(bw.pos / 8));
      for (int r = 0; r < h; r++)
        for (int c = 0; c < w; c++)
          patch[r * w + c] = plane[(uint64_t)(y0 + r) * W + (x0 + c)];

      /* Stage 1, custom Paeth filter: the first row is skipped
       * (C5: the first row of every patch); for the others the residual is the
       * pixel minus the selected neighbour of the row above, mod 256 (C1);
       * missing neighbours at the patch's columns 0 and w-1 are replaced by
       * Top (C4). */
      for (int c = 0; c < w; c++) resid[c] = patch[c];
      for (int r = 1; r < h; r++) {
        for (int c = 0; c < w; c++) {
          int pred;
          if (predictor == 0) {
            int t = patch[(r - 1) * w + c];
            int tl = c > 0 ? patch[(r - 1) * w + c - 1] : t;
            int tr = c < w - 1 ? patch[(r - 1) * w + c + 1] : t;
            pred = l3ref_predict(tl, t, tr);
          } else {   /* original Paeth: left, top, top-left of the SAME patch (0 when absent) */
            int a = c > 0 ? patch[r * w + c - 1] : 0;
            int b = patch[(r - 1) * w + c];
            int cc = c > 0 ? patch[(r - 1) * w + c - 1] : 0;
            pred = l3ref_predict_png(a, b, cc);
          }
          resid[r * w + c] = (uint8_t)((patch[r * w + c] - pred) & 0xFF);
        }
      }

      /* Stage 2, base-delta per row: "the first four bits
       * represent the number of bits per delta for each row, and the following
       * eight bits the base value. Then, the deltas of the row ... are
       * appended. All the rows are concatenated" */
      for (int r = 0; r < h; r++) {
        int k, base;
        l3ref_bd_encode_row(resid + r * w, w, r == 0, base_rule, k_extra, &k, &base, deltas);
        bw_put(&bw, (uint32_t)k, 4);
        bw_put(&bw, (uint32_t)base, 8);
        for (int c = 0; c < w; c++) bw_put(&bw, deltas[c], k);
      }
      bw.pos = (bw.pos + 7) & ~7ull;                      /* byte-align the patch (C8) */
      if (bw.pos > bw.cap_bits) bw.overflow = 1;
    }
  }
  free(patch); free(resid); free(deltas);
  if (bw.overflow) return 0;
  return hdr + bw.pos / 8;
}

/* ------------------------------------------------------------------------ */
/* Decoder                                     */
/* ------------------------------------------------------------------------ */

typedef struct {
  uint32_t W, H;
  int N;
  uint64_t gx, gy, P;
  uint64_t hdr, data_len;
  const uint8_t* data;
  int predictor;   /* 0 custom (L3IF), 1 original Paeth (L3IP, ablation variant) */
} l3hdr;

/* Reading a1 / C9: header parse and validation order:
 *   magic -> UNRECOGNIZED_FORMAT; short header, W/H/N zero, shape mismatch,
 *   offsets table outside the file, offsets not starting at 0 / not strictly
 *   increasing over R||G||B / not inside the data section -> CORRUPT_HEADER. */
static int parse_header_v_(const uint8_t* f, uint64_t len, uint32_t exp_W, uint32_t exp_H, l3hdr* h,
                           int allow_variant);
static int parse_header_(const uint8_t* f, uint64_t len, uint32_t exp_W, uint32_t exp_H, l3hdr* h) {
  return parse_header_v_(f, len, exp_W, exp_H, h, 0);
}
static int parse_header_v_(const uint8_t* f, uint64_t len, uint32_t exp_W, uint32_t exp_H, l3hdr* h,
                           int allow_variant) {
  h->predictor = 0;
  if (len >= 4 && allow_variant && memcmp(f, "L3IP", 4) == 0) h->predictor = 1;
  else if (len < 4 || memcmp(f, "L3IF", 4) != 0) return L3REF_E_UNRECOGNIZED_FORMAT;
  if (len < 13) return L3REF_E_CORRUPT_HEADER;
  h->W = get_u32le_(f + 4);
  h->H = get_u32le_(f + 8);
  h->N = f[12];
  if (h->W == 0 || h->H == 0 || h->N == 0) return L3REF_E_CORRUPT_HEADER;
  if ((exp_W && h->W != exp_W) || (exp_H && h->H != exp_H)) return L3REF_E_CORRUPT_HEADER;
  h->gx = ceil_div_(h->W, (uint64_t)h->N);
  h->gy = ceil_div_(h->H, (uint64_t)h->N);
  h->P = h->gx * h->gy;
  h->hdr = 13ull + 12ull * h->P;
  if (len < h->hdr) return L3REF_E_CORRUPT_HEADER;
  h->data = f + h->hdr;
  h->data_len = len - h->hdr;
  uint64_t prev = 0;
  for (uint64_t u = 0; u < 3 * h->P; u++) {
    uint64_t o = get_u32le_(f + 13 + 4 * u);
    if (u == 0 && o != 0) return L3REF_E_CORRUPT_HEADER;
    if (u > 0 && o <= prev) return L3REF_E_CORRUPT_HEADER;
    if (o >= h->data_len) return L3REF_E_CORRUPT_HEADER;
    prev = o;
  }
  return L3REF_OK;
}

/* Decode unit u = ch*P + p into the planar output (pitch W). */
static int decode_unit_(const l3hdr* h, const uint8_t* file, uint64_t u, uint8_t* out) {
  uint64_t ch = u / h->P, p = u % h->P;
  uint64_t start = get_u32le_(file + 13 + 4 * u);
  uint64_t end = (u + 1 < 3 * h->P) ? get_u32le_(file + 13 + 4 * (u + 1)) : h->data_len;
  uint64_t px = p % h->gx, py = p / h->gx;
  int N = h->N;
  uint64_t x0 = px * N, y0 = py * N;
  int w = (int)((h->W - x0) < (uint64_t)N ? (h->W - x0) : (uint64_t)N);
  int hh = (int)((h->H - y0) < (uint64_t)N ? (h->H - y0) : (uint64_t)N);
  uint8_t* plane = out + ch * (uint64_t)h->W * h->H;

  bitreader br = {h->data + start, (end - start) * 8ull, 0};
  uint8_t res[256];
  for (int r = 0; r < hh; r++) {
    /* "the decoder first reads the four bits as well as the following eight
     * bits to identify the number of bits per entry and the base value for the
     * row (Step 1). From this point, the decoder extracts the delta one by one
     * and adds the base value to reconstruct the original value (Step 2)."
     * (PAPER.md:152). Reading C6: k outside 1..8 is a corrupt stream. */
    uint32_t k, base, d;
    if (!br_get(&br, 4, &k)) return L3REF_E_TRUNCATED_STREAM;
    if (k < 1 || k > 8) return L3REF_E_CORRUPT_STREAM;
    if (!br_get(&br, 8, &base)) return L3REF_E_TRUNCATED_STREAM;
    for (int c = 0; c < w; c++) {
      if (!br_get(&br, (int)k, &d)) return L3REF_E_TRUNCATED_STREAM;
      res[c] = (uint8_t)((base + d) & 0xFF);             /* C7: wraps mod 256 */
    }
    uint8_t* row = plane + (y0 + r) * h->W + x0;
    if (r == 0) {
      /* "the first row is stored in a raw data format" */
      for (int c = 0; c < w; c++) row[c] = res[c];
    } else {
      /* "The reference value can be computed by inspecting the three
       * neighboring pixels in the preceding row ... Then we add the stored
       * residual ... to the pixel value" */
      const uint8_t* up = row - h->W;
      for (int c = 0; c < w; c++) {
        if (h->predictor == 0) {
          int t = up[c];
          int tl = c > 0 ? up[c - 1] : t;
          int tr = c < w - 1 ? up[c + 1] : t;
          row[c] = (uint8_t)((l3ref_predict(tl, t, tr) + res[c]) & 0xFF);
        } else {   /* original Paeth: depends on the pixel just decoded to the left */
          int a = c > 0 ? row[c - 1] : 0;
          int cc = c > 0 ? up[c - 1] : 0;
          row[c] = (uint8_t)((l3ref_predict_png(a, up[c], cc) + res[c]) & 0xFF);
        }
      }
    }
  }
  /* trailing padding / bytes after the last row are ignored */
  return L3REF_OK;
}

static int decode_image_(const uint8_t* file, uint64_t len, uint32_t exp_W, uint32_t exp_H, uint8_t* out,
                         uint64_t out_cap, int64_t* bad_unit, uint32_t* W, uint32_t* H, int* N, uint64_t* P,
                         int allow_variant);

int l3ref_decode_image(const uint8_t* file, uint64_t len, uint32_t exp_W, uint32_t exp_H,
                       uint8_t* out, uint64_t out_cap, int64_t* bad_unit,
                       uint32_t* W, uint32_t* H, int* N, uint64_t* P) {
  return decode_image_(file, len, exp_W, exp_H, out, out_cap, bad_unit, W, H, N, P, 0);
}

/* Accepts both "L3IF" and the ablation variant "L3IP" (original Paeth). */
int l3ref_decode_image_variant(const uint8_t* file, uint64_t len, uint8_t* out, uint64_t out_cap,
                               uint32_t* W, uint32_t* H) {
  return decode_image_(file, len, 0, 0, out, out_cap, NULL, W, H, NULL, NULL, 1);
}

static int decode_image_(const uint8_t* file, uint64_t len, uint32_t exp_W, uint32_t exp_H, uint8_t* out,
                         uint64_t out_cap, int64_t* bad_unit, uint32_t* W, uint32_t* H, int* N, uint64_t* P,
                         int allow_variant) {
  l3hdr h;
  memset(&h, 0, sizeof h);
  if (bad_unit) *bad_unit = -1;
  int st = parse_header_v_(file, len, exp_W, exp_H, &h, allow_variant);
  if (W) *W = h.W;
  if (H) *H = h.H;
  if (N) *N = h.N;
  if (P) *P = h.P;
  if (st != L3REF_OK) return st;
  if (out_cap < 3ull * h.W * h.H) return L3REF_E_INVALID_ARGUMENT;
  /* units in canonical order: channel R, G, B; patches row-major (C9) */
  for (uint64_t u = 0; u < 3 * h.P; u++) {
    st = decode_unit_(&h, file, u, out);
    if (st != L3REF_OK) {
      if (bad_unit) *bad_unit = (int64_t)u;
      return st;
    }
  }
  return L3REF_OK;
}

/* ------------------------------------------------------------------------ */
/* Batch decode over a pthread pool                        */
/* ------------------------------------------------------------------------ */

typedef struct {
  const uint8_t* src;
  const uint64_t* src_offsets;
  const int32_t* shapes;
  int n;
  uint8_t* out;
  const uint64_t* out_offsets;
  l3hdr* hdrs;
  int32_t* status;
  int64_t* first_bad;   /* per image, minimum failing unit (atomic) */
  int32_t* bad_code;    /* code belonging to first_bad */
  uint64_t* unit_prefix;
  uint64_t total_units;
  uint64_t next;        /* job counter (atomic) */
  pthread_mutex_t mu;
} batch_ctx;

static void* batch_worker_(void* arg) {
  batch_ctx* b = (batch_ctx*)arg;
  for (;;) {
    uint64_t j = __atomic_fetch_add(&b->next, 1, __ATOMIC_RELAXED);
    if (j >= b->total_units) break;
    int i = 0;                                   /* image of job j (linear search: small n) */
    while (b->unit_prefix[i + 1] <= j) i++;
    if (b->status[i] != L3REF_OK) continue;      /* header failed: no units */
    uint64_t u = j - b->unit_prefix[i];
    int st = decode_unit_(&b->hdrs[i], b->src + b->src_offsets[i], u, b->out + b->out_offsets[i]);
    if (st != L3REF_OK) {
      pthread_mutex_lock(&b->mu);
      if (b->first_bad[i] < 0 || (int64_t)u < b->first_bad[i]) {
        b->first_bad[i] = (int64_t)u;
        b->bad_code[i] = st;
      }
      pthread_mutex_unlock(&b->mu);
    }
  }
  return NULL;
}

void l3ref_decode_batch(const uint8_t* src, const uint64_t* src_offsets, const int32_t* shapes,
                        int n, uint8_t* out, const uint64_t* out_offsets,
                        int32_t* status, int32_t* bad_unit, int threads) {
  batch_ctx b;
  memset(&b, 0, sizeof b);
  b.src = src; b.src_offsets = src_offsets; b.shapes = shapes; b.n = n;
  b.out = out; b.out_offsets = out_offsets; b.status = status;
  b.hdrs = (l3hdr*)calloc((size_t)n + 1, sizeof(l3hdr));
  b.first_bad = (int64_t*)malloc(sizeof(int64_t) * ((size_t)n + 1));
  b.bad_code = (int32_t*)calloc((size_t)n + 1, sizeof(int32_t));
  b.unit_prefix = (uint64_t*)calloc((size_t)n + 1, sizeof(uint64_t));
  pthread_mutex_init(&b.mu, NULL);
  for (int i = 0; i < n; i++) {
    b.first_bad[i] = -1;
    status[i] = parse_header_(src + src_offsets[i], src_offsets[i + 1] - src_offsets[i],
                              (uint32_t)shapes[2 * i + 1], (uint32_t)shapes[2 * i], &b.hdrs[i]);
    b.unit_prefix[i + 1] = b.unit_prefix[i] + (status[i] == L3REF_OK ? 3 * b.hdrs[i].P : 0);
  }
  b.total_units = b.unit_prefix[n];
  if (threads < 1) threads = 1;
  if (threads == 1) {
    batch_worker_(&b);
  } else {
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
    for (int t = 0; t < threads; t++) pthread_create(&th[t], NULL, batch_worker_, &b);
    for (int t = 0; t < threads; t++) pthread_join(th[t], NULL);
    free(th);
  }
  for (int i = 0; i < n; i++) {
    if (bad_unit) bad_unit[i] = -1;
    if (status[i] == L3REF_OK && b.first_bad[i] >= 0) {
      status[i] = b.bad_code[i];
      if (bad_unit) bad_unit[i] = (int32_t)b.first_bad[i];
    }
  }
  pthread_mutex_destroy(&b.mu);
  free(b.hdrs); free(b.first_bad); free(b.bad_code); free(b.unit_prefix);
}

/* ------------------------------------------------------------------------ */
/* Normalisation definition (reading C14), fp64                              */
/* ------------------------------------------------------------------------ */

void l3ref_normalize(const uint8_t* x, uint64_t count_per_channel, int channels,
                     const double* mean, const double* std, double* y) {
  for (int c = 0; c < channels; c++)
    for (uint64_t i = 0; i < count_per_channel; i++) {
      uint64_t j = (uint64_t)c * count_per_channel + i;
      y[j] = ((double)x[j] / 255.0 - mean[c]) / std[c];
    }
}
