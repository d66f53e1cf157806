/*
 * ranger_oracle.c -- TEST INFRASTRUCTURE ONLY (see oracle.h).
 *
 * Plain-C restatement of the reference census template-matching path of
 * arxiv/paper_2604_07980 (proj/include/ranger/, cited below as file:line).
 * It is the checker the CUDA path is compared against; it is pinned to the
 * reference itself by tests/test_oracle_cpu.py (against oracle/_ref when the
 * reference is present, and against the committed tests/golden fixtures
 * generated from it).  Scalar, single-threaded, written for clarity.
 *
 * Build: gcc -std=c11 -O2 -ffp-contract=off -fPIC -shared (oracle/Makefile).
 * No FMA contraction, so every double expression rounds exactly as the
 * reference's (x86-64 SSE2) build does.
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "oracle.h"

/* ======================================================== census */

/* census.hpp:43-56: sentinel 1, then 25 window compares, window row -2 first,
 * column -2 first, each shifted in at the LSB; 0 if the window leaves. */
static uint32_t census_at(const uint8_t* img, int w, int h, int sx, int sy) {
  if (sx < 2 || sy < 2 || sx >= w - 2 || sy >= h - 2) return 0u;
  const uint8_t centre = img[(size_t)sy * w + sx];
  uint32_t code = 1u;
  for (int dy = -2; dy <= 2; ++dy) {
    const uint8_t* row = img + (size_t)(sy + dy) * w + sx;
    for (int dx = -2; dx <= 2; ++dx) code = (code << 1) | (uint32_t)(row[dx] > centre);
  }
  return code;
}

/* 9x7 extension: census.hpp:43-56 with rows -3..3, columns
 * -4..4; 63 compares after the sentinel, which ends in bit 63. */
static uint64_t census_at64(const uint8_t* img, int w, int h, int sx, int sy) {
  if (sx < 4 || sy < 3 || sx >= w - 4 || sy >= h - 3) return 0u;
  const uint8_t centre = img[(size_t)sy * w + sx];
  uint64_t code = 1u;
  for (int dy = -3; dy <= 3; ++dy) {
    const uint8_t* row = img + (size_t)(sy + dy) * w + sx;
    for (int dx = -4; dx <= 4; ++dx) code = (code << 1) | (uint64_t)(row[dx] > centre);
  }
  return code;
}

/* census.hpp:59-64 detail::scaled_coords */
static void scaled_coords(int out, int src, int* m) {
  for (int i = 0; i < out; ++i)
    m[i] = (out == src) ? i : (int)lround((double)i * (double)src / (double)out);
}

/* census.hpp:69-86 */
int orc_census_transform(const uint8_t* img, int w, int h, int ow, int oh, uint32_t* out) {
  if (ow > w || oh > h) return RG_EINVAL;
  if (ow < 1 || oh < 1) return RG_EINVAL;
  int* mx = (int*)malloc(sizeof(int) * (size_t)ow);
  int* my = (int*)malloc(sizeof(int) * (size_t)oh);
  scaled_coords(ow, w, mx);
  scaled_coords(oh, h, my);
  for (int y = 0; y < oh; ++y)
    for (int x = 0; x < ow; ++x) out[(size_t)y * ow + x] = census_at(img, w, h, mx[x], my[y]);
  free(mx);
  free(my);
  return RG_OK;
}

int orc_census_transform64(const uint8_t* img, int w, int h, int ow, int oh, uint64_t* out) {
  if (ow > w || oh > h || ow < 1 || oh < 1) return RG_EINVAL;
  int* mx = (int*)malloc(sizeof(int) * (size_t)ow);
  int* my = (int*)malloc(sizeof(int) * (size_t)oh);
  scaled_coords(ow, w, mx);
  scaled_coords(oh, h, my);
  for (int y = 0; y < oh; ++y)
    for (int x = 0; x < ow; ++x) out[(size_t)y * ow + x] = census_at64(img, w, h, mx[x], my[y]);
  free(mx);
  free(my);
  return RG_OK;
}

/* census.hpp:100-138.  The reference merges per-row x-intervals of the
 * clipped rectangles; the set of computed pixels is exactly the union of the
 * clipped rectangles, which is what the mask below marks. */
int orc_census_transform_rois(const uint8_t* img, int w, int h, int ow, int oh,
                              const rg_rect* rois, int n_rois, uint32_t* out) {
  if (ow > w || oh > h) return RG_EINVAL;
  if (ow < 1 || oh < 1) return RG_EINVAL; /* CensusImage(ow, oh) needs ow*oh >= 0 */
  int* mx = (int*)malloc(sizeof(int) * (size_t)ow);
  int* my = (int*)malloc(sizeof(int) * (size_t)oh);
  unsigned char* mask = (unsigned char*)calloc((size_t)ow * oh, 1);
  scaled_coords(ow, w, mx);
  scaled_coords(oh, h, my);
  for (int r = 0; r < n_rois; ++r) {
    const int x0 = rois[r].x0 > 0 ? rois[r].x0 : 0;
    const int x1 = rois[r].x1 < ow ? rois[r].x1 : ow;
    const int y0 = rois[r].y0 > 0 ? rois[r].y0 : 0;
    const int y1 = rois[r].y1 < oh ? rois[r].y1 : oh;
    if (x0 >= x1) continue;
    for (int y = y0; y < y1; ++y) memset(mask + (size_t)y * ow + x0, 1, (size_t)(x1 - x0));
  }
  for (int y = 0; y < oh; ++y)
    for (int x = 0; x < ow; ++x)
      out[(size_t)y * ow + x] = mask[(size_t)y * ow + x] ? census_at(img, w, h, mx[x], my[y]) : 0u;
  free(mask);
  free(mx);
  free(my);
  return RG_OK;
}

/* ======================================================== matcher */

typedef struct {
  const uint32_t* codes;
  int w, h;
  const uint64_t* codes64; /* 9x7 extension: used when non-NULL */
} raster;

static int r_inside(const raster* r, int x, int y) { return x >= 0 && x < r->w && y >= 0 && y < r->h; }
static uint64_t r_code(const raster* r, int x, int y) {
  return r->codes64 ? r->codes64[(size_t)y * r->w + x] : r->codes[(size_t)y * r->w + x];
}

/* census.hpp:167-171 */
static double subpixel(double cm, double c0, double cp) {
  const double denom = cm + cp - 2.0 * c0;
  if (denom <= 0.0) return 0.0;
  return -(cp - cm) / (2.0 * denom);
}

/* census.hpp:178-272 block_match.  Returns RG_EINVAL for an empty range on a
 * non-empty block; res->has_value = 0 encodes std::nullopt. */
static int block_match(const int32_t* pts, int np, rg_search_range rg, const raster* L,
                       const raster* R, rg_match_result* res) {
  memset(res, 0, sizeof(*res));
  res->cost_minus = -1.0;
  res->cost_plus = -1.0;
  if (np == 0) return RG_OK; /* :181 nullopt before the range check */
  if (rg.dx_min > rg.dx_max || rg.dy_min > rg.dy_max) return RG_EINVAL; /* :182-183 */
  const int ndx = rg.dx_max - rg.dx_min + 1, ndy = rg.dy_max - rg.dy_min + 1;
  const size_t nc = (size_t)ndx * ndy;
  double* mean = (double*)malloc(sizeof(double) * nc);
  int* cnt = (int*)calloc(nc, sizeof(int));
  int* vx = (int*)malloc(sizeof(int) * (size_t)np);
  int* vy = (int*)malloc(sizeof(int) * (size_t)np);
  uint64_t* lc = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)np);
  int nv = 0;
  /* :195-201 keep points whose left descriptor exists */
  for (int k = 0; k < np; ++k) {
    const int x = pts[2 * k], y = pts[2 * k + 1];
    if (!r_inside(L, x, y)) continue;
    const uint64_t c = r_code(L, x, y);
    if (c == 0u) continue;
    vx[nv] = x;
    vy[nv] = y;
    lc[nv] = c;
    ++nv;
  }
  /* :203-223 mean Hamming cost per offset over contributing points */
  for (int iy = 0; iy < ndy; ++iy) {
    const int dy = rg.dy_min + iy;
    for (int ix = 0; ix < ndx; ++ix) {
      const int dx = rg.dx_min + ix;
      long sum = 0;
      int n = 0;
      for (int k = 0; k < nv; ++k) {
        const int rx = vx[k] - dx, ry = vy[k] + dy;
        if (!r_inside(R, rx, ry)) continue;
        const uint64_t rc = r_code(R, rx, ry);
        if (rc == 0u) continue;
        sum += __builtin_popcountll(lc[k] ^ rc);
        ++n;
      }
      mean[(size_t)iy * ndx + ix] = n > 0 ? (double)sum / n : INFINITY;
      cnt[(size_t)iy * ndx + ix] = n;
    }
  }
  /* :225-252 argmin of (mean, |dx|, dy, dx) */
  int bix = -1, biy = -1;
  double best = INFINITY;
  for (int iy = 0; iy < ndy; ++iy) {
    const int dy = rg.dy_min + iy;
    for (int ix = 0; ix < ndx; ++ix) {
      const int dx = rg.dx_min + ix;
      const double c = mean[(size_t)iy * ndx + ix];
      if (c == INFINITY) continue;
      int take = c < best;
      if (!take && c == best && bix >= 0) {
        const int bdx = rg.dx_min + bix, bdy = rg.dy_min + biy;
        const int adx = abs(dx), abdx = abs(bdx);
        take = adx < abdx || (adx == abdx && (dy < bdy || (dy == bdy && dx < bdx)));
      }
      if (take) {
        best = c;
        bix = ix;
        biy = iy;
      }
    }
  }
  if (bix >= 0) {
    /* :255-270 result + sub-pixel when the winner is interior in dx */
    res->has_value = 1;
    res->dx_int = rg.dx_min + bix;
    res->dy_int = rg.dy_min + biy;
    res->cost = best;
    res->valid_points = cnt[(size_t)biy * ndx + bix];
    res->dx_subpix = (double)res->dx_int;
    if (bix > 0 && bix + 1 < ndx) {
      const double cm = mean[(size_t)biy * ndx + bix - 1];
      const double cp = mean[(size_t)biy * ndx + bix + 1];
      if (cm != INFINITY && cp != INFINITY) {
        res->cost_minus = cm;
        res->cost_plus = cp;
        res->dx_subpix = res->dx_int + subpixel(cm, best, cp);
      }
    }
  }
  free(mean);
  free(cnt);
  free(vx);
  free(vy);
  free(lc);
  return RG_OK;
}

/* census.hpp:281-303 forward_backward_match */
static int fb_match(const int32_t* pts, int np, rg_search_range rg, double tau_v,
                    const raster* L, const raster* R, rg_match_result* res) {
  int st = block_match(pts, np, rg, L, R, res);
  if (st != RG_OK || !res->has_value) return st;
  int32_t* back = (int32_t*)malloc(sizeof(int32_t) * 2 * (size_t)np);
  for (int k = 0; k < np; ++k) {
    back[2 * k] = pts[2 * k] - res->dx_int;
    back[2 * k + 1] = pts[2 * k + 1] + res->dy_int;
  }
  rg_search_range brg = {-rg.dx_max, -rg.dx_min, -res->dy_int, -res->dy_int};
  rg_match_result bwd;
  st = block_match(back, np, brg, R, L, &bwd);
  free(back);
  res->verified = 0;
  if (st == RG_OK && bwd.has_value) {
    const double dx_v = res->dx_subpix + bwd.dx_subpix;
    res->verified = fabs(dx_v) < tau_v;
  }
  return st;
}

/* census.hpp:307-315 batch_match (and plain block_match for mode 0) */
int orc_match_blocks(const uint32_t* left, int lw, int lh, const uint32_t* right, int rw,
                     int rh, const int32_t* points_xy, const int64_t* offsets,
                     const rg_search_range* ranges, int n_blocks, int mode, double tau_v,
                     rg_match_result* out) {
  const raster L = {left, lw, lh, NULL}, R = {right, rw, rh, NULL};
  for (int b = 0; b < n_blocks; ++b) {
    const int np = (int)(offsets[b + 1] - offsets[b]);
    const int32_t* p = points_xy + 2 * offsets[b];
    const int st = mode == RG_MATCH_FWD_BWD ? fb_match(p, np, ranges[b], tau_v, &L, &R, &out[b])
                                            : block_match(p, np, ranges[b], &L, &R, &out[b]);
    if (st != RG_OK) return st;
  }
  return RG_OK;
}

int orc_match_blocks64(const uint64_t* left, int lw, int lh, const uint64_t* right, int rw, int rh,
                       const int32_t* points_xy, const int64_t* offsets, const rg_search_range* ranges,
                       int n_blocks, int mode, double tau_v, rg_match_result* out) {
  const raster L = {NULL, lw, lh, left}, R = {NULL, rw, rh, right};
  for (int b = 0; b < n_blocks; ++b) {
    const int np = (int)(offsets[b + 1] - offsets[b]);
    const int32_t* p = points_xy + 2 * offsets[b];
    const int st = mode == RG_MATCH_FWD_BWD ? fb_match(p, np, ranges[b], tau_v, &L, &R, &out[b])
                                            : block_match(p, np, ranges[b], &L, &R, &out[b]);
    if (st != RG_OK) return st;
  }
  return RG_OK;
}

/* ======================================================== object ranger */

/* template_match.hpp:48-61 validate(RangerConfig) */
static int validate_cfg(const rg_ranger_config* c) {
  if (c->tau_s <= 0 || c->tau_d <= 0 || c->tau_v < 0) return RG_EINVAL;
  if (c->n_min < 1 || c->close_scale < 1) return RG_EINVAL;
  if (c->grid_side_points < 1 || c->max_total_points < 1 || c->close_block_side_points < 1)
    return RG_EINVAL;
  if (c->max_objects < 0 || c->dx_max_far < 0 || c->dx_max_close < 0) return RG_EINVAL;
  return RG_OK;
}

/* detection.hpp:23-30 to_pixel_box */
typedef struct {
  double x0, y0, x1, y1;
} pbox;
static pbox to_pixel_box(const rg_detection* d, int w, int h) {
  pbox b;
  b.x0 = (d->cx - d->w / 2) * w;
  b.x1 = (d->cx + d->w / 2) * w;
  b.y0 = (d->cy - d->h / 2) * h;
  b.y1 = (d->cy + d->h / 2) * h;
  return b;
}
static int pbox_contains(const pbox* b, double x, double y) {
  return x >= b->x0 && x < b->x1 && y >= b->y0 && y < b->y1; /* detection.hpp:19-21 */
}

/* template_match.hpp:63-67 */
static int classify(const rg_detection* d, int w, int h, double tau_s) {
  const double a = d->w * w, b = d->h * h;
  return (a > b ? a : b) < tau_s ? RG_KIND_FAR : RG_KIND_CLOSE;
}

/* template_match.hpp:71-89: j occludes i iff positive overlap and lower bottom */
static int occludes(const rg_detection* di, const rg_detection* dj) {
  const double ix0 = di->cx - di->w / 2, ix1 = di->cx + di->w / 2;
  const double iy0 = di->cy - di->h / 2, iy1 = di->cy + di->h / 2;
  const double jx0 = dj->cx - dj->w / 2, jx1 = dj->cx + dj->w / 2;
  const double jy0 = dj->cy - dj->h / 2, jy1 = dj->cy + dj->h / 2;
  const double ox = (ix1 < jx1 ? ix1 : jx1) - (ix0 > jx0 ? ix0 : jx0);
  const double oy = (iy1 < jy1 ? iy1 : jy1) - (iy0 > jy0 ? iy0 : jy0);
  return ox > 0 && oy > 0 && jy1 > iy1;
}

int orc_find_occluders(const rg_detection* dets, int n, int32_t* occ_offsets, int32_t* occ_idx) {
  int k = 0;
  for (int i = 0; i < n; ++i) {
    occ_offsets[i] = k;
    for (int j = 0; j < n; ++j)
      if (j != i && occludes(&dets[i], &dets[j])) occ_idx[k++] = j;
  }
  occ_offsets[n] = k;
  return RG_OK;
}

/* template_match.hpp:94-114 select_objects: frontal by area desc, rest by
 * bottom desc, ties by id (index as a final, reference-unspecified tiebreak) */
static const rg_detection* g_sel_dets;
static int cmp_frontal(const void* a, const void* b) {
  const int i = *(const int*)a, j = *(const int*)b;
  const rg_detection *di = &g_sel_dets[i], *dj = &g_sel_dets[j];
  const double ai = di->w * di->h, aj = dj->w * dj->h;
  if (ai != aj) return ai > aj ? -1 : 1;
  if (di->id != dj->id) return di->id < dj->id ? -1 : 1;
  return i - j;
}
static int cmp_rest(const void* a, const void* b) {
  const int i = *(const int*)a, j = *(const int*)b;
  const rg_detection *di = &g_sel_dets[i], *dj = &g_sel_dets[j];
  const double bi = di->cy + di->h / 2, bj = dj->cy + dj->h / 2;
  if (bi != bj) return bi > bj ? -1 : 1;
  if (di->id != dj->id) return di->id < dj->id ? -1 : 1;
  return i - j;
}
int orc_select_objects(const rg_detection* dets, int n, const rg_ranger_config* cfg,
                       int32_t* out_idx, int* n_out) {
  int* fr = (int*)malloc(sizeof(int) * (size_t)(n + 1));
  int* rs = (int*)malloc(sizeof(int) * (size_t)(n + 1));
  int nf = 0, nr = 0;
  for (int i = 0; i < n; ++i) {
    const double cx = dets[i].cx, cy = dets[i].cy; /* template_match.hpp:28-30 */
    const int frontal = cx >= cfg->crop_x0 && cx < cfg->crop_x1 && cy >= cfg->crop_y0 && cy < cfg->crop_y1;
    if (frontal)
      fr[nf++] = i;
    else
      rs[nr++] = i;
  }
  g_sel_dets = dets;
  qsort(fr, (size_t)nf, sizeof(int), cmp_frontal);
  qsort(rs, (size_t)nr, sizeof(int), cmp_rest);
  int m = 0;
  for (int i = 0; i < nf && m < cfg->max_objects; ++i) out_idx[m++] = fr[i];
  for (int i = 0; i < nr && m < cfg->max_objects; ++i) out_idx[m++] = rs[i];
  *n_out = m;
  free(fr);
  free(rs);
  return RG_OK;
}

/* template_match.hpp:155-223 sample_query_points */
int orc_sample_query_points(const rg_detection* det, int kind, const double* occ_boxes,
                            int n_occ, const rg_ranger_config* cfg, int w, int h,
                            int64_t* block_offsets, int32_t* points_xy,
                            rg_search_range* ranges, int cap_blocks, int64_t cap_points,
                            int* n_blocks) {
  const pbox box = to_pixel_box(det, w, h);
  const double bw = box.x1 - box.x0, bh = box.y1 - box.y0;
  int cap = (int)sqrt((double)cfg->max_total_points);
  if (cap < 1) cap = 1;
  int nb = 0;
  int64_t np = 0;
  block_offsets[0] = 0;
#define OCCLUDED(fx, fy)                                                         \
  ({                                                                             \
    int _o = 0;                                                                  \
    for (int _k = 0; _k < n_occ && !_o; ++_k) {                                  \
      const pbox _b = {occ_boxes[4 * _k], occ_boxes[4 * _k + 1],                 \
                       occ_boxes[4 * _k + 2], occ_boxes[4 * _k + 3]};            \
      _o = pbox_contains(&_b, (fx), (fy));                                       \
    }                                                                            \
    _o;                                                                          \
  })
  if (kind == RG_KIND_FAR) {
    const int n = cfg->grid_side_points < cap ? cfg->grid_side_points : cap;
    const int64_t start = np;
    for (int j = 0; j < n; ++j) {
      const double fy = box.y0 + (j + 0.5) * bh / n;
      for (int i = 0; i < n; ++i) {
        const double fx = box.x0 + (i + 0.5) * bw / n;
        const int px = (int)lround(fx), py = (int)lround(fy);
        if (px < 0 || px >= w || py < 0 || py >= h) continue;
        if (OCCLUDED(fx, fy)) continue;
        if (np >= cap_points) return RG_EOVERFLOW;
        points_xy[2 * np] = px;
        points_xy[2 * np + 1] = py;
        ++np;
      }
    }
    if (np - start >= 4) {
      if (nb >= cap_blocks) return RG_EOVERFLOW;
      ranges[nb].dx_min = 0;
      ranges[nb].dx_max = cfg->dx_max_far;
      ranges[nb].dy_min = -1;
      ranges[nb].dy_max = 1;
      block_offsets[++nb] = np;
    } else {
      np = start;
    }
    *n_blocks = nb;
    return RG_OK;
  }
  const int s = cfg->close_scale;
  const int cw = w / s, ch = h / s;
  const double half_tau = cfg->tau_s / 2;
  int cols = (int)(bw / half_tau), rows = (int)(bh / half_tau);
  if (cols < 2) cols = 2;
  if (rows < 2) rows = 2;
  const int q = cfg->close_block_side_points < cap ? cfg->close_block_side_points : cap;
  const int dx_max_scaled = (cfg->dx_max_close + s - 1) / s;
  for (int r = 0; r < rows; ++r) {
    for (int c = 0; c < cols; ++c) {
      const double sx0 = box.x0 + c * bw / cols;
      const double sy0 = box.y0 + r * bh / rows;
      const double sw = bw / cols, sh = bh / rows;
      const int64_t start = np;
      for (int j = 0; j < q; ++j) {
        const double fy = sy0 + (j + 0.5) * sh / q;
        for (int i = 0; i < q; ++i) {
          const double fx = sx0 + (i + 0.5) * sw / q;
          if (fx < 0 || fx >= w || fy < 0 || fy >= h) continue;
          if (OCCLUDED(fx, fy)) continue;
          const int mx = (int)lround(fx * cw / (double)w);
          const int my = (int)lround(fy * ch / (double)h);
          if (mx < 0 || mx >= cw || my < 0 || my >= ch) continue;
          if (np >= cap_points) return RG_EOVERFLOW;
          points_xy[2 * np] = mx;
          points_xy[2 * np + 1] = my;
          ++np;
        }
      }
      if (np - start >= 4) {
        if (nb >= cap_blocks) return RG_EOVERFLOW;
        ranges[nb].dx_min = 0;
        ranges[nb].dx_max = dx_max_scaled;
        ranges[nb].dy_min = -1;
        ranges[nb].dy_max = 1;
        block_offsets[++nb] = np;
      } else {
        np = start;
      }
    }
  }
#undef OCCLUDED
  *n_blocks = nb;
  return RG_OK;
}

/* template_match.hpp:126-148 aggregate_close_disparities */
static int cmp_double(const void* a, const void* b) {
  const double x = *(const double*)a, y = *(const double*)b;
  return x < y ? -1 : (x > y ? 1 : 0);
}
int orc_aggregate_close_disparities(const double* disps, int n, double tau_d, int n_min,
                                    int32_t* valid, double* disparity, int32_t* run_length) {
  *valid = 0;
  *disparity = 0;
  *run_length = 0;
  if (n == 0) return RG_OK;
  double* v = (double*)malloc(sizeof(double) * (size_t)n);
  memcpy(v, disps, sizeof(double) * (size_t)n);
  qsort(v, (size_t)n, sizeof(double), cmp_double);
  int best_start = -1, best_len = 0, start = 0;
  for (int i = 1; i <= n; ++i) {
    if (i == n || v[i] - v[i - 1] >= tau_d) {
      const int len = i - start;
      if (len >= best_len) { /* later (larger-disparity) run wins ties */
        best_len = len;
        best_start = start;
      }
      start = i;
    }
  }
  if (best_len >= n_min) {
    *valid = 1;
    *run_length = best_len;
    *disparity = v[best_start + best_len / 2];
  }
  free(v);
  return RG_OK;
}

/* template_match.hpp:245-253 detail::add_roi */
static rg_rect roi_of(pbox b, double sx, double sy, int dil_x, int dil_y, int w, int h) {
  rg_rect r;
  const int x0 = (int)floor(b.x0 * sx) - dil_x, x1 = (int)ceil(b.x1 * sx) + dil_x + 1;
  const int y0 = (int)floor(b.y0 * sy) - dil_y, y1 = (int)ceil(b.y1 * sy) + dil_y + 1;
  r.x0 = x0 > 0 ? x0 : 0;
  r.x1 = x1 < w ? x1 : w;
  r.y0 = y0 > 0 ? y0 : 0;
  r.y1 = y1 < h ? y1 : h;
  return r;
}

static int cmp_int(const void* a, const void* b) { return *(const int32_t*)a - *(const int32_t*)b; }

/* template_match.hpp:260-363 estimate_object_disparities (ROI census, as the
 * reference runs it), plus geometry.hpp:142-146 range when focal/baseline > 0 */
int orc_estimate_object_disparities(const uint8_t* left, const uint8_t* right, int w, int h,
                                    const rg_detection* dets, int n, const rg_ranger_config* cfg,
                                    rg_census_cache* cache, double focal_px, double baseline_m,
                                    rg_object_disparity* out, int* n_out, rg_ranger_stats* stats) {
  if (validate_cfg(cfg) != RG_OK) return RG_EINVAL;
  if (cfg->census_9x7 && cache) return RG_EINVAL; /* caches hold 5x5 codes */
  *n_out = 0;
  if (stats) {
    stats->query_points = 0;
    stats->image_pixels = (int64_t)w * h;
    stats->n_far = stats->n_close = 0;
  }
  if (n == 0) return RG_OK;
  int32_t* sel = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
  int nsel = 0;
  orc_select_objects(dets, n, cfg, sel, &nsel);
  qsort(sel, (size_t)nsel, sizeof(int32_t), cmp_int); /* :278 input order */
  int32_t* occ_off = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n + 1));
  int32_t* occ_idx = (int32_t*)malloc(sizeof(int32_t) * (size_t)n * (size_t)n + 1);
  orc_find_occluders(dets, n, occ_off, occ_idx);

  const int s = cfg->close_scale, cw = w / s, ch = h / s;
  const int dx_max_scaled = (cfg->dx_max_close + s - 1) / s;
  /* per selected object: its blocks (CSR over all blocks of the frame) */
  int cap_blocks = 0;
  for (int t = 0; t < nsel; ++t) {
    const pbox b = to_pixel_box(&dets[sel[t]], w, h);
    int cols = (int)((b.x1 - b.x0) / (cfg->tau_s / 2)), rows = (int)((b.y1 - b.y0) / (cfg->tau_s / 2));
    cap_blocks += (cols < 2 ? 2 : cols) * (rows < 2 ? 2 : rows) + 1;
  }
  int64_t cap_pts = (int64_t)cap_blocks * cfg->max_total_points + 1;
  int64_t* boff = (int64_t*)malloc(sizeof(int64_t) * (size_t)(cap_blocks + 1));
  int64_t* tmpoff = (int64_t*)malloc(sizeof(int64_t) * (size_t)(cap_blocks + 1));
  int32_t* pts = (int32_t*)malloc(sizeof(int32_t) * 2 * (size_t)cap_pts);
  rg_search_range* rgs = (rg_search_range*)malloc(sizeof(rg_search_range) * (size_t)(cap_blocks + 1));
  int* owner = (int*)malloc(sizeof(int) * (size_t)(cap_blocks + 1));
  int* kind = (int*)malloc(sizeof(int) * (size_t)n);
  rg_rect* far_rois = (rg_rect*)malloc(sizeof(rg_rect) * (size_t)(nsel + 1));
  rg_rect* sc_rois = (rg_rect*)malloc(sizeof(rg_rect) * (size_t)(nsel + 1));
  int n_far_roi = 0, n_sc_roi = 0, nb = 0;
  boff[0] = 0;
  double* occ_boxes = (double*)malloc(sizeof(double) * 4 * (size_t)(n + 1));
  for (int t = 0; t < nsel; ++t) {
    const int i = sel[t];
    kind[i] = classify(&dets[i], w, h, cfg->tau_s);
    int no = 0;
    for (int k = occ_off[i]; k < occ_off[i + 1]; ++k) {
      const pbox ob = to_pixel_box(&dets[occ_idx[k]], w, h);
      occ_boxes[4 * no] = ob.x0;
      occ_boxes[4 * no + 1] = ob.y0;
      occ_boxes[4 * no + 2] = ob.x1;
      occ_boxes[4 * no + 3] = ob.y1;
      ++no;
    }
    int got = 0;
    orc_sample_query_points(&dets[i], kind[i], occ_boxes, no, cfg, w, h, tmpoff,
                            pts + 2 * boff[nb], rgs + nb, cap_blocks - nb, cap_pts - boff[nb], &got);
    /* sample_query_points wrote offsets relative to its own start */
    for (int k = 1; k <= got; ++k) boff[nb + k] = boff[nb] + tmpoff[k];
    for (int k = 0; k < got; ++k) owner[nb + k] = i;
    if (stats) stats->query_points += boff[nb + got] - boff[nb];
    nb += got;
    const pbox box = to_pixel_box(&dets[i], w, h);
    if (kind[i] == RG_KIND_FAR) {
      if (stats) ++stats->n_far;
      far_rois[n_far_roi++] = roi_of(box, 1, 1, cfg->dx_max_far + 2, 3, w, h);
    } else {
      if (stats) ++stats->n_close;
      sc_rois[n_sc_roi++] = roi_of(box, (double)cw / w, (double)ch / h, dx_max_scaled + 2, 3, cw, ch);
    }
  }
  /* split blocks by kind, keeping order (:297-300) */
  int n_far_b = 0, n_close_b = 0;
  for (int b = 0; b < nb; ++b) {
    if (kind[owner[b]] == RG_KIND_FAR)
      ++n_far_b;
    else
      ++n_close_b;
  }

  uint32_t *fl = NULL, *fr = NULL, *sl = NULL, *sr = NULL;
  int own_full = 0, own_scaled = 0;
  if (cache && cache->has_full) {
    fl = cache->full_left;
    fr = cache->full_right;
  } else if (n_far_b > 0 && !cfg->census_9x7) {
    fl = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)w * h);
    fr = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)w * h);
    orc_census_transform_rois(left, w, h, w, h, far_rois, n_far_roi, fl);
    orc_census_transform_rois(right, w, h, w, h, far_rois, n_far_roi, fr);
    if (cache) {
      memcpy(cache->full_left, fl, sizeof(uint32_t) * (size_t)w * h);
      memcpy(cache->full_right, fr, sizeof(uint32_t) * (size_t)w * h);
      cache->has_full = 1;
    }
    own_full = 1;
  }
  if (cache && cache->has_scaled) {
    sl = cache->scaled_left;
    sr = cache->scaled_right;
  } else if (n_close_b > 0 && !cfg->census_9x7) {
    sl = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)cw * ch);
    sr = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)cw * ch);
    orc_census_transform_rois(left, w, h, cw, ch, sc_rois, n_sc_roi, sl);
    orc_census_transform_rois(right, w, h, cw, ch, sc_rois, n_sc_roi, sr);
    if (cache) {
      memcpy(cache->scaled_left, sl, sizeof(uint32_t) * (size_t)cw * ch);
      memcpy(cache->scaled_right, sr, sizeof(uint32_t) * (size_t)cw * ch);
      cache->has_scaled = 1;
    }
    own_scaled = 1;
  }
  rg_match_result* res = (rg_match_result*)calloc((size_t)(nb + 1), sizeof(rg_match_result));
  raster FL = {fl, w, h, NULL}, FR = {fr, w, h, NULL}, SL = {sl, cw, ch, NULL}, SR = {sr, cw, ch, NULL};
  uint64_t *f64l = NULL, *f64r = NULL, *s64l = NULL, *s64r = NULL;
  if (cfg->census_9x7) { /* extension: full-frame 9x7 rasters (same results as ROI rasters) */
    f64l = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)w * h);
    f64r = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)w * h);
    s64l = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)cw * ch + 8);
    s64r = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)cw * ch + 8);
    orc_census_transform64(left, w, h, w, h, f64l);
    orc_census_transform64(right, w, h, w, h, f64r);
    if (cw > 0 && ch > 0) {
      orc_census_transform64(left, w, h, cw, ch, s64l);
      orc_census_transform64(right, w, h, cw, ch, s64r);
    }
    FL.codes64 = f64l;
    FR.codes64 = f64r;
    SL.codes64 = s64l;
    SR.codes64 = s64r;
  }
  for (int b = 0; b < nb; ++b) {
    const int far = kind[owner[b]] == RG_KIND_FAR;
    fb_match(pts + 2 * boff[b], (int)(boff[b + 1] - boff[b]), rgs[b], cfg->tau_v,
             far ? &FL : &SL, far ? &FR : &SR, &res[b]);
  }
  /* :332-361 results in input order */
  double* disps = (double*)malloc(sizeof(double) * (size_t)(nb + 1));
  for (int t = 0; t < nsel; ++t) {
    const int i = sel[t];
    rg_object_disparity od;
    memset(&od, 0, sizeof(od));
    od.det_id = dets[i].id;
    od.kind = kind[i];
    if (kind[i] == RG_KIND_FAR) {
      for (int b = 0; b < nb; ++b) {
        if (owner[b] != i) continue;
        if (res[b].has_value && res[b].verified) {
          od.valid = 1;
          od.disparity = res[b].dx_subpix;
          od.n_blocks_used = 1;
        }
        break;
      }
    } else {
      int nd = 0;
      for (int b = 0; b < nb; ++b)
        if (owner[b] == i && res[b].has_value && res[b].verified) disps[nd++] = res[b].dx_subpix * s;
      int32_t v, rl;
      double d;
      orc_aggregate_close_disparities(disps, nd, cfg->tau_d, cfg->n_min, &v, &d, &rl);
      od.valid = v;
      od.disparity = d;
      od.n_blocks_used = rl;
    }
    /* geometry.hpp:142-146 with canonical Q (:124-127): z = f / ((1/b) d) */
    if (od.valid && od.disparity > 0 && focal_px > 0 && baseline_m > 0) od.z_cam = focal_px / ((1.0 / baseline_m) * od.disparity);
    out[(*n_out)++] = od;
  }
  free(disps);
  free(res);
  free(f64l);
  free(f64r);
  free(s64l);
  free(s64r);
  if (own_full) {
    free(fl);
    free(fr);
  }
  if (own_scaled) {
    free(sl);
    free(sr);
  }
  free(occ_boxes);
  free(far_rois);
  free(sc_rois);
  free(kind);
  free(owner);
  free(rgs);
  free(pts);
  free(boff);
  free(tmpoff);
  free(occ_off);
  free(occ_idx);
  free(sel);
  return RG_OK;
}

/* ======================================================== BM / autorect */

#define RAW_INVALID (-32768) /* image.hpp:52-56 DisparityMap::kInvalid */

/* bm.hpp:24-32 */
static int validate_bm(const rg_bm_params* p) {
  if (p->block_size < 3 || p->block_size % 2 == 0) return RG_EINVAL;
  if (p->num_disparities < 1) return RG_EINVAL;
  if (p->uniqueness_ratio < 0) return RG_EINVAL;
  if (p->downscale < 1) return RG_EINVAL;
  return RG_OK;
}

/* bm.hpp:37-106 bm_disparity_at_scale (crop-local coordinates) */
static void bm_at_scale(const uint8_t* L, const uint8_t* R, int w, int h, int nd, int bs,
                        int dmin, double tex, double uniq, int16_t* out) {
  const int hw = bs / 2, d_lo = dmin, d_hi = dmin + nd;
  long* sad = (long*)malloc(sizeof(long) * (size_t)nd);
  for (size_t i = 0; i < (size_t)w * h; ++i) out[i] = RAW_INVALID;
  for (int y = hw; y < h - hw; ++y) {
    for (int x = hw; x < w - hw; ++x) {
      long grad = 0; /* texture gate: horizontal |diffs| in the window */
      for (int j = -hw; j <= hw; ++j) {
        const uint8_t* r = L + (size_t)(y + j) * w + x;
        for (int i = -hw; i < hw; ++i) grad += labs((long)r[i + 1] - (long)r[i]);
      }
      if (grad < tex) continue;
      int n_eval = 0;
      for (int d = d_lo; d < d_hi; ++d) {
        const int idx = d - d_lo;
        if (x - d - hw < 0 || x - d + hw >= w) {
          sad[idx] = -1;
          continue;
        }
        long s = 0;
        for (int j = -hw; j <= hw; ++j) {
          const uint8_t* lr = L + (size_t)(y + j) * w + x;
          const uint8_t* rr = R + (size_t)(y + j) * w + x - d;
          for (int i = -hw; i <= hw; ++i) s += labs((long)lr[i] - (long)rr[i]);
        }
        sad[idx] = s;
        ++n_eval;
      }
      if (n_eval == 0) continue;
      int bi = -1;
      long best = 0x7fffffffffffffffL;
      for (int i = 0; i < nd; ++i)
        if (sad[i] >= 0 && sad[i] < best) {
          best = sad[i];
          bi = i;
        }
      long second = 0x7fffffffffffffffL;
      for (int i = 0; i < nd; ++i)
        if (sad[i] >= 0 && abs(i - bi) > 1 && sad[i] < second) second = sad[i];
      if (second != 0x7fffffffffffffffL && (double)best * (1.0 + uniq / 100.0) >= (double)second)
        continue;
      double d_hat = d_lo + bi;
      if (bi > 0 && bi + 1 < nd && sad[bi - 1] >= 0 && sad[bi + 1] >= 0)
        d_hat += subpixel((double)sad[bi - 1], (double)best, (double)sad[bi + 1]);
      long raw = lround(d_hat * 16);
      const long lo = (long)d_lo * 16, hi = (long)d_hi * 16 - 1;
      raw = raw < lo ? lo : (raw > hi ? hi : raw);
      out[(size_t)y * w + x] = (int16_t)raw;
    }
  }
  free(sad);
}

/* image.hpp:98-116 downscale */
static void downscale(const uint8_t* in, int w, int h, int s, uint8_t* out) {
  const int ow = w / s, oh = h / s;
  for (int y = 0; y < oh; ++y)
    for (int x = 0; x < ow; ++x) {
      int sum = 0;
      for (int j = 0; j < s; ++j)
        for (int i = 0; i < s; ++i) sum += in[(size_t)(y * s + j) * w + x * s + i];
      out[(size_t)y * ow + x] = (uint8_t)lround(sum / (double)(s * s));
    }
}

/* bm.hpp:113-135 bm_disparity (+ image.hpp:122-141 upscale_disparity) */
int orc_bm_disparity(const uint8_t* left, const uint8_t* right, int w, int h, const rg_bm_params* p,
                     int16_t* out) {
  if (validate_bm(p) != RG_OK) return RG_EINVAL;
  const int s = p->downscale;
  if (s == 1) {
    bm_at_scale(left, right, w, h, p->num_disparities, p->block_size, p->min_disparity,
                p->texture_threshold, p->uniqueness_ratio, out);
    return RG_OK;
  }
  const int ow = w / s, oh = h / s;
  if (ow < 1 || oh < 1) return RG_EINVAL; /* image.hpp:104 */
  const int qmin = (p->min_disparity + s - 1) / s;
  int qn = (p->min_disparity + p->num_disparities) / s - qmin;
  if (qn < 1) qn = 1;
  uint8_t* dl = (uint8_t*)malloc((size_t)ow * oh);
  uint8_t* dr = (uint8_t*)malloc((size_t)ow * oh);
  int16_t* dm = (int16_t*)malloc(sizeof(int16_t) * (size_t)ow * oh);
  downscale(left, w, h, s, dl);
  downscale(right, w, h, s, dr);
  bm_at_scale(dl, dr, ow, oh, qn, p->block_size, qmin, p->texture_threshold, p->uniqueness_ratio, dm);
  for (size_t i = 0; i < (size_t)w * h; ++i) out[i] = RAW_INVALID;
  const int lo = qmin * 16 * s;
  for (int y = 0; y < oh; ++y)
    for (int x = 0; x < ow; ++x) {
      const int r = dm[(size_t)y * ow + x];
      int v = RAW_INVALID;
      if (r != RAW_INVALID) {
        const int scaled = r * s;
        if (scaled >= lo && scaled <= 32767) v = scaled;
      }
      for (int j = 0; j < s; ++j)
        for (int i = 0; i < s; ++i) out[(size_t)(y * s + j) * w + x * s + i] = (int16_t)v;
    }
  free(dl);
  free(dr);
  free(dm);
  return RG_OK;
}

/* autorect.hpp:22-58 auto_rect_search (+ image.hpp:145-154 shift_vertical,
 * image.hpp:75-82 crop) */
int orc_auto_rect_search(const uint8_t* left, const uint8_t* right, int w, int h, const rg_rect* roi,
                         int delta_min, int delta_max, const rg_bm_params* p, int32_t* best_delta,
                         int64_t* counts) {
  const int rw = roi->x1 - roi->x0, rh = roi->y1 - roi->y0;
  if (rw < p->block_size || rh < p->block_size) return RG_EINVAL;
  if (roi->x0 < 0 || roi->y0 < 0 || roi->x1 > w || roi->y1 > h) return RG_EINVAL;
  if (delta_min > delta_max) return RG_EINVAL;
  if (validate_bm(p) != RG_OK) return RG_EINVAL;
  uint8_t* lc = (uint8_t*)malloc((size_t)rw * rh);
  uint8_t* rc = (uint8_t*)malloc((size_t)rw * rh);
  int16_t* d = (int16_t*)malloc(sizeof(int16_t) * (size_t)rw * rh);
  for (int y = 0; y < rh; ++y) memcpy(rc + (size_t)y * rw, right + (size_t)(roi->y0 + y) * w + roi->x0, (size_t)rw);
  int best = 0;
  long best_count = -1;
  for (int delta = delta_min; delta <= delta_max; ++delta) {
    for (int y = 0; y < rh; ++y) {
      int sy = roi->y0 + y - delta; /* shift_vertical: out(y) = in(clamp(y - dy)) */
      sy = sy < 0 ? 0 : (sy >= h ? h - 1 : sy);
      memcpy(lc + (size_t)y * rw, left + (size_t)sy * w + roi->x0, (size_t)rw);
    }
    orc_bm_disparity(lc, rc, rw, rh, p, d);
    long count = 0;
    const int lo = p->min_disparity * 16;
    for (size_t i = 0; i < (size_t)rw * rh; ++i)
      if (d[i] != RAW_INVALID && d[i] > lo) ++count;
    if (counts) counts[delta - delta_min] = count;
    int better = count > best_count;
    if (count == best_count)
      better = abs(delta) < abs(best) || (abs(delta) == abs(best) && delta < best);
    if (better) {
      best_count = count;
      best = delta;
    }
  }
  *best_delta = best;
  free(lc);
  free(rc);
  free(d);
  return RG_OK;
}

/* ======================================================== SGM (8f row 2) */

/* sgm.hpp:37-56 sgm_cost_volume: popcount of the census XOR, 27 where the
 * right column leaves the frame */
static void sgm_cost(const uint32_t* cl, const uint32_t* cr, int w, int h, int nd, int d_lo, uint8_t* cost) {
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x) {
      uint8_t* c = cost + ((size_t)y * w + x) * nd;
      for (int i = 0; i < nd; ++i) {
        const int rx = x - (d_lo + i);
        c[i] = (rx < 0 || rx >= w) ? 27 : (uint8_t)__builtin_popcount(cl[(size_t)y * w + x] ^ cr[(size_t)y * w + rx]);
      }
    }
}

/* sgm.hpp:60-110 one directional pass, restated path by path (each path is
 * walked from the pixel whose predecessor leaves the image) */
int orc_sgm_direction_pass(const uint8_t* cost, int w, int h, int nd, int p1, int p2, int sx, int sy,
                           int32_t* acc) {
  const int big = 0x7fffffff / 4;
  int32_t* L = (int32_t*)malloc(sizeof(int32_t) * (size_t)nd);
  int32_t* Ln = (int32_t*)malloc(sizeof(int32_t) * (size_t)nd);
  for (int y0 = 0; y0 < h; ++y0)
    for (int x0 = 0; x0 < w; ++x0) {
      const int px = x0 - sx, py = y0 - sy;
      if (px >= 0 && px < w && py >= 0 && py < h) continue; /* not a path start */
      int x = x0, y = y0, first = 1, pmin = 0;
      while (x >= 0 && x < w && y >= 0 && y < h) {
        const uint8_t* c = cost + ((size_t)y * w + x) * nd;
        int mn = big;
        for (int d = 0; d < nd; ++d) {
          if (first) {
            Ln[d] = c[d];
          } else {
            int best = L[d];
            if (d > 0 && L[d - 1] + p1 < best) best = L[d - 1] + p1;
            if (d + 1 < nd && L[d + 1] + p1 < best) best = L[d + 1] + p1;
            if (pmin + p2 < best) best = pmin + p2;
            Ln[d] = c[d] + best - pmin;
          }
          if (Ln[d] < mn) mn = Ln[d];
        }
        int32_t* a = acc + ((size_t)y * w + x) * nd;
        for (int d = 0; d < nd; ++d) {
          a[d] += Ln[d];
          L[d] = Ln[d];
        }
        pmin = mn;
        first = 0;
        x += sx;
        y += sy;
      }
    }
  free(L);
  free(Ln);
  return RG_OK;
}

/* sgm.hpp:118-155 */
int orc_sgm_disparity(const uint8_t* left, const uint8_t* right, int w, int h, int nd, int d_lo, int p1, int p2,
                      int16_t* out) {
  if (nd < 1 || p1 < 0 || p2 < p1) return RG_EINVAL;
  uint32_t* cl = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)w * h);
  uint32_t* cr = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)w * h);
  orc_census_transform(left, w, h, w, h, cl);
  orc_census_transform(right, w, h, w, h, cr);
  uint8_t* cost = (uint8_t*)malloc((size_t)w * h * nd);
  sgm_cost(cl, cr, w, h, nd, d_lo, cost);
  int32_t* acc = (int32_t*)calloc((size_t)w * h * nd, sizeof(int32_t));
  const int dirs[4][2] = {{1, 0}, {0, 1}, {1, 1}, {-1, 1}};
  for (int k = 0; k < 4; ++k) orc_sgm_direction_pass(cost, w, h, nd, p1, p2, dirs[k][0], dirs[k][1], acc);
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x) {
      const int32_t* a = acc + ((size_t)y * w + x) * nd;
      int bi = -1;
      int32_t best = 0x7fffffff;
      for (int i = 0; i < nd; ++i) {
        const int rx = x - (d_lo + i);
        if (rx < 0 || rx >= w) continue;
        if (a[i] < best) {
          best = a[i];
          bi = i;
        }
      }
      int16_t r = (int16_t)-32768;
      if (bi >= 0) {
        double d_hat = d_lo + bi;
        if (bi > 0 && bi + 1 < nd && x - (d_lo + bi + 1) >= 0) d_hat += subpixel((double)a[bi - 1], (double)best, (double)a[bi + 1]);
        long v = lround(d_hat * 16.0);
        const long lo = (long)d_lo * 16, hi = (long)(d_lo + nd) * 16 - 1;
        v = v < lo ? lo : (v > hi ? hi : v);
        r = (int16_t)v;
      }
      out[(size_t)y * w + x] = r;
    }
  free(cl);
  free(cr);
  free(cost);
  free(acc);
  return RG_OK;
}

/* ======================================================== dense BM objects (8f row 3) */

/* pipeline.hpp:304-328 box_disparity + geometry.hpp:162-178 dynamic_disparity_variance */
int orc_box_disparity(const int16_t* raw, int w, int h, const rg_detection* dets, int n, double sigma_obs2,
                      double gamma, double sigma_sys2, rg_box_stats* out) {
  for (int b = 0; b < n; ++b) {
    const rg_detection* d = &dets[b];
    const double bx0 = (d->cx - d->w / 2) * w, bx1 = (d->cx + d->w / 2) * w;
    const double by0 = (d->cy - d->h / 2) * h, by1 = (d->cy + d->h / 2) * h;
    int y0 = (int)floor(by0), y1 = (int)ceil(by1), x0 = (int)floor(bx0), x1 = (int)ceil(bx1);
    if (y0 < 0) y0 = 0;
    if (x0 < 0) x0 = 0;
    if (y1 > h) y1 = h;
    if (x1 > w) x1 = w;
    const int bw = x1 > x0 ? x1 - x0 : 0, bh = y1 > y0 ? y1 - y0 : 0;
    double* v = (double*)malloc(sizeof(double) * ((size_t)bw * bh + 1));
    size_t m = 0;
    for (int y = y0; y < y1; ++y)
      for (int x = x0; x < x1; ++x) {
        const int16_t r = raw[(size_t)y * w + x];
        if (r != -32768) v[m++] = r / 16.0;
      }
    rg_box_stats o = {0, 0, 0.0, 0.0};
    if (m > 0) {
      qsort(v, m, sizeof(double), cmp_double);
      const size_t near_from = (3 * (m - 1)) / 4;
      double sn = 0, sa = 0;
      for (size_t i = near_from; i < m; ++i) sn += v[i];
      for (size_t i = 0; i < m; ++i) sa += v[i];
      const double mean_near = sn / (double)(m - near_from), mean_all = sa / (double)m;
      const double diff = mean_near - mean_all;
      o.valid = 1;
      o.count = (int32_t)m;
      o.median = v[(m - 1) / 2];
      o.variance = sigma_obs2 / (double)(m - near_from) + gamma * diff * diff + sigma_sys2;
    }
    out[b] = o;
    free(v);
  }
  return RG_OK;
}
