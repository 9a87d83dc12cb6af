/*
 * lmgs oracle — CPU float64 restatement of the reference 3DGS forward path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library, and
 * only as the checker (or the timed CPU baseline), never as the product path.
 *
 * Reference (all paths under /root/reference/pkg/src/landmark/):
 *   project_splats    gaussian_core.py:187-230   -> oracle_project
 *   quat_to_rotmat    gaussian_core.py:93-102
 *   covariance_3d     gaussian_core.py:105-117
 *   eval_sh_colors    gaussian_core.py:129-142   (degree <= 1, reference semantics)
 *   rasterize         gaussian_core.py:340-403   -> oracle_bin / oracle_blend
 *   _sort_order       gaussian_core.py:277-283   (lexsort by (depth, prim_id))
 *   _blend            gaussian_core.py:286-332
 *
 * Floating-point restatement (probed against torch 2.11 CPU / MKL in this
 * image):
 *   * means @ r_wc.T and j @ r_wc are MKL dgemm: fma(a2,b2, fma(a1,b1, a0*b0));
 *   * the covariance and cov2d products are torch bmm: ((a0*b0 + a1*b1) + a2*b2);
 *   * `camera.fx / z` is torch's scalar/tensor = reciprocal(z) * fx;
 *   * quats.norm is a sequential sum of squares then sqrt;
 *   * torch.sqrt (MKL VML, HA mode) is NOT correctly rounded (<= 1 ulp low on
 *     ~0.7% of inputs); this file uses IEEE sqrt, so radius / lam_max may sit
 *     1 ulp above the reference's.  The tile predicates are insensitive at
 *     that scale (margins are certified by oracle_margins()).
 * This file is compiled with -ffp-contract=off so no other FMA is formed.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define TERM_EPS 1e-4
#define SIGMA_MAX 0.9999
#define COV2D_REG 0.3
#define NEAR_CULL_Z 0.01
static const double SH_C0 = 0.28209479177387814;
static const double SH_C1 = 0.4886025119029199;
static const double SH_C2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
                                -1.0925484305920792, 0.5462742152960396};
static const double SH_C3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658,
                                0.3731763325901154, -0.4570457994644658, 1.445305721320277,
                                -0.5900435899266435};

typedef struct {
  double r_wc[9], t_wc[3], center[3];
  double fx, fy, cx, cy, lim_x, lim_y;
  int64_t width, height;
} ocam_t;

int oracle_abi_version(void) { return 3; }

/* ------------------------------------------------------------------------ */
/* projection: gaussian_core.py:187-230 (+ eval_sh_colors 129-142)           */

static double mkl_dot3(double a0, double b0, double a1, double b1, double a2, double b2) {
  return fma(a2, b2, fma(a1, b1, a0 * b0));
}
static double bmm_dot3(double a0, double b0, double a1, double b1, double a2, double b2) {
  return (a0 * b0 + a1 * b1) + a2 * b2;
}

/* colour for one Gaussian.  eval_deg <= 1 is the reference's eval_sh_colors
 * (gaussian_core.py:129-142); eval_deg 2/3 extend it with the standard real SH
 * basis in the same sign convention, still clamp(.,0,1) with no +0.5 offset. */
static void sh_color(const float* sh, int64_t ncoef, int eval_deg, const float* mean,
                     const double* center, double* out) {
  double d0 = (double)mean[0] - center[0], d1 = (double)mean[1] - center[1],
         d2 = (double)mean[2] - center[2];
  double nrm = sqrt((d0 * d0 + d1 * d1) + d2 * d2);
  if (nrm < 1e-12) nrm = 1e-12;
  double x = d0 / nrm, y = d1 / nrm, z = d2 / nrm;
  for (int ch = 0; ch < 3; ch++) {
    double c = SH_C0 * (double)sh[0 * 3 + ch];
    if (eval_deg >= 1 && ncoef >= 4) {
      c = ((c - (SH_C1 * y) * (double)sh[1 * 3 + ch]) + (SH_C1 * z) * (double)sh[2 * 3 + ch]) -
          (SH_C1 * x) * (double)sh[3 * 3 + ch];
    }
    if (eval_deg >= 2 && ncoef >= 9) {
      double xx = x * x, yy = y * y, zz = z * z, xy = x * y, yz = y * z, xz = x * z;
      c = c + SH_C2[0] * xy * (double)sh[4 * 3 + ch] + SH_C2[1] * yz * (double)sh[5 * 3 + ch] +
          SH_C2[2] * (2.0 * zz - xx - yy) * (double)sh[6 * 3 + ch] +
          SH_C2[3] * xz * (double)sh[7 * 3 + ch] + SH_C2[4] * (xx - yy) * (double)sh[8 * 3 + ch];
      if (eval_deg >= 3 && ncoef >= 16) {
        c = c + SH_C3[0] * y * (3.0 * xx - yy) * (double)sh[9 * 3 + ch] +
            SH_C3[1] * xy * z * (double)sh[10 * 3 + ch] +
            SH_C3[2] * y * (4.0 * zz - xx - yy) * (double)sh[11 * 3 + ch] +
            SH_C3[3] * z * (2.0 * zz - 3.0 * xx - 3.0 * yy) * (double)sh[12 * 3 + ch] +
            SH_C3[4] * x * (4.0 * zz - xx - yy) * (double)sh[13 * 3 + ch] +
            SH_C3[5] * z * (xx - yy) * (double)sh[14 * 3 + ch] +
            SH_C3[6] * x * (xx - 3.0 * yy) * (double)sh[15 * 3 + ch];
      }
    }
    out[ch] = c < 0.0 ? 0.0 : (c > 1.0 ? 1.0 : c);
  }
}

/* Per input Gaussian i (0..n-1): kept[i] = z > 0.01; for kept ones the
 * projected geometry.  Returns M = number kept.  cov2d = (a, b, c) with
 * b = cov2d[0,1] as the reference reads it (gaussian_core.py:223, 309). */
int64_t oracle_project(int64_t n, const float* means, const float* quats, const float* scales,
                       const float* logits, const float* sh, int64_t ncoef, int64_t eval_deg,
                       const ocam_t* cam, uint8_t* kept, double* mean2d, double* cov2d,
                       double* depth, double* radius, double* color, double* opac) {
  int64_t m = 0;
  const double* R = cam->r_wc;
  const double* t = cam->t_wc;
#pragma omp parallel for reduction(+ : m) schedule(static)
  for (int64_t i = 0; i < n; i++) {
    const float* mu = means + 3 * i;
    double p[3];
    for (int j = 0; j < 3; j++)
      p[j] = mkl_dot3((double)mu[0], R[3 * j + 0], (double)mu[1], R[3 * j + 1], (double)mu[2],
                      R[3 * j + 2]) + t[j];
    double x = p[0], y = p[1], z = p[2];
    kept[i] = z > NEAR_CULL_Z;
    if (!kept[i]) continue;
    m++;
    mean2d[2 * i + 0] = cam->fx * x / z + cam->cx;
    mean2d[2 * i + 1] = cam->fy * y / z + cam->cy;
    depth[i] = z;
    /* quat_to_rotmat (93-102) */
    const float* q = quats + 4 * i;
    double qw = q[0], qx = q[1], qy = q[2], qz = q[3];
    double nr = sqrt(((qw * qw + qx * qx) + qy * qy) + qz * qz);
    double w = qw / nr, X = qx / nr, Y = qy / nr, Z = qz / nr;
    double r[9] = {1 - 2 * (Y * Y + Z * Z), 2 * (X * Y - w * Z), 2 * (X * Z + w * Y),
                   2 * (X * Y + w * Z), 1 - 2 * (X * X + Z * Z), 2 * (Y * Z - w * X),
                   2 * (X * Z - w * Y), 2 * (Y * Z + w * X), 1 - 2 * (X * X + Y * Y)};
    /* covariance_3d (105-117): m = R * s[None, :], cov = m m^T */
    const float* s = scales + 3 * i;
    double M[9], C[9];
    for (int a = 0; a < 3; a++)
      for (int b = 0; b < 3; b++) M[3 * a + b] = r[3 * a + b] * (double)s[b];
    for (int a = 0; a < 3; a++)
      for (int b = 0; b < 3; b++)
        C[3 * a + b] = bmm_dot3(M[3 * a], M[3 * b], M[3 * a + 1], M[3 * b + 1], M[3 * a + 2],
                                M[3 * b + 2]);
    /* Jacobian with the clamped off-axis angle (205-218) */
    double tx = fmin(fmax(x / z, -cam->lim_x), cam->lim_x) * z;
    double ty = fmin(fmax(y / z, -cam->lim_y), cam->lim_y) * z;
    double rz = 1.0 / z;
    double J[6] = {rz * cam->fx, 0.0, -cam->fx * tx / (z * z),
                   0.0, rz * cam->fy, -cam->fy * ty / (z * z)};
    double JW[6], T1[6], C2[4];
    for (int a = 0; a < 2; a++)
      for (int b = 0; b < 3; b++)
        JW[3 * a + b] = mkl_dot3(J[3 * a], R[b], J[3 * a + 1], R[3 + b], J[3 * a + 2], R[6 + b]);
    for (int a = 0; a < 2; a++)
      for (int b = 0; b < 3; b++)
        T1[3 * a + b] =
            bmm_dot3(JW[3 * a], C[b], JW[3 * a + 1], C[3 + b], JW[3 * a + 2], C[6 + b]);
    for (int a = 0; a < 2; a++)
      for (int b = 0; b < 2; b++)
        C2[2 * a + b] = bmm_dot3(T1[3 * a], JW[3 * b], T1[3 * a + 1], JW[3 * b + 1],
                                 T1[3 * a + 2], JW[3 * b + 2]);
    double ca = C2[0] + COV2D_REG, cb = C2[1], cc = C2[3] + COV2D_REG;
    cov2d[3 * i + 0] = ca;
    cov2d[3 * i + 1] = cb;
    cov2d[3 * i + 2] = cc;
    double h = 0.5 * (ca - cc);
    double lam = 0.5 * (ca + cc) + sqrt(h * h + cb * cb);
    radius[i] = 3.0 * sqrt(lam);
    opac[i] = 1.0 / (1.0 + exp(-(double)logits[i]));
    sh_color(sh + i * ncoef * 3, ncoef, (int)eval_deg, mu, cam->center, color + 3 * i);
  }
  return m;
}

/* ------------------------------------------------------------------------ */
/* tile overlap predicate, rasterize 362-373:                                */
/*   s in tile (tx,ty,tw,th) iff hi_x >= tx & lo_x <= tx+tw & hi_y >= ty &   */
/*   lo_y <= ty+th, lo/hi = mean2d -/+ radius (fp64), tw = min(ts, W - tx).  */
/* Restated as an inclusive index range with exact comparisons.              */

static void axis_range(double lo, double hi, int64_t size, int64_t ts, int64_t* a, int64_t* b) {
  int64_t nt = (size + ts - 1) / ts;
  /* first tile j with lo <= min((j+1)*ts, size) */
  int64_t j;
  if (!(lo > -2.0 * (double)ts)) j = 0; /* also catches NaN */
  else if (lo > (double)size + 2.0 * ts) j = nt;
  else {
    j = (int64_t)floor(lo / (double)ts) - 2;
    if (j < 0) j = 0;
  }
  while (j < nt) {
    int64_t end = (j + 1) * ts < size ? (j + 1) * ts : size;
    if (lo <= (double)end) break;
    j++;
  }
  /* last tile k with k*ts <= hi */
  int64_t k;
  if (!(hi < (double)size + 2.0 * ts)) k = nt - 1;
  else if (hi < -2.0 * (double)ts) k = -1;
  else {
    k = (int64_t)floor(hi / (double)ts) + 2;
    if (k > nt - 1) k = nt - 1;
  }
  while (k >= 0 && !((double)(k * ts) <= hi)) k--;
  *a = j;
  *b = k;
}

/* brute-force form of the same predicate, exactly as the reference writes it */
static int overlap_brute(double lox, double hix, double loy, double hiy, int64_t tx, int64_t ty,
                         int64_t tw, int64_t th) {
  return (hix >= (double)tx) & (lox <= (double)(tx + tw)) & (hiy >= (double)ty) &
         (loy <= (double)(ty + th));
}

typedef struct {
  double depth;
  int64_t pid;
  int64_t idx;
} okey_t;

static int cmp_key(const void* a, const void* b) {
  const okey_t* x = (const okey_t*)a;
  const okey_t* y = (const okey_t*)b;
  if (x->depth < y->depth) return -1;
  if (x->depth > y->depth) return 1;
  if (x->pid < y->pid) return -1;
  if (x->pid > y->pid) return 1;
  return 0;
}

/* Bin splats into tiles.  Splat arrays are the compacted kept splats (M).
 * counts[T] must be zeroed by the caller.  Pass 1 (lists == NULL): fill
 * counts, return K.  Pass 2: `offsets` = exclusive scan of counts (T+1);
 * fills lists[K] with splat indices, each tile's list in (depth, prim_id)
 * order, i.e. TileRecord.order (gaussian_core.py:392 -> _sort_order 277-283).
 * brute != 0 evaluates the reference's per-tile mask literally (O(T*M)). */
int64_t oracle_bin(int64_t m, const double* mean2d, const double* radius, const double* depth,
                   const int64_t* prim_id, int64_t width, int64_t height, int64_t ts, int brute,
                   int64_t* counts, const int64_t* offsets, int64_t* lists) {
  int64_t tx_n = (width + ts - 1) / ts, ty_n = (height + ts - 1) / ts;
  int64_t ntiles = tx_n * ty_n;
  okey_t* order = (okey_t*)malloc(sizeof(okey_t) * (m > 0 ? m : 1));
  for (int64_t i = 0; i < m; i++) {
    order[i].depth = depth[i];
    order[i].pid = prim_id[i];
    order[i].idx = i;
  }
  qsort(order, (size_t)m, sizeof(okey_t), cmp_key);
  int64_t total = 0;
  if (brute) {
    /* reference loop order: tiles row-major, each tile scans all splats in
     * global (depth, pid) order -> identical to per-tile lexsort. */
    int64_t* fill = NULL;
    for (int64_t tyi = 0; tyi < ty_n; tyi++)
      for (int64_t txi = 0; txi < tx_n; txi++) {
        int64_t t = tyi * tx_n + txi;
        int64_t tx = txi * ts, ty = tyi * ts;
        int64_t tw = ts < width - tx ? ts : width - tx, th = ts < height - ty ? ts : height - ty;
        int64_t c = 0;
        for (int64_t r = 0; r < m; r++) {
          int64_t i = order[r].idx;
          double mx = mean2d[2 * i], my = mean2d[2 * i + 1], rr = radius[i];
          if (overlap_brute(mx - rr, mx + rr, my - rr, my + rr, tx, ty, tw, th)) {
            if (lists) lists[offsets[t] + c] = i;
            c++;
          }
        }
        if (!lists) counts[t] = c;
        total += c;
      }
    (void)fill;
    free(order);
    return total;
  }
  int64_t* cursor = NULL;
  if (lists) {
    cursor = (int64_t*)malloc(sizeof(int64_t) * (ntiles > 0 ? ntiles : 1));
    for (int64_t t = 0; t < ntiles; t++) cursor[t] = offsets[t];
  }
  for (int64_t r = 0; r < m; r++) {
    int64_t i = order[r].idx;
    double mx = mean2d[2 * i], my = mean2d[2 * i + 1], rr = radius[i];
    int64_t x0, x1, y0, y1;
    axis_range(mx - rr, mx + rr, width, ts, &x0, &x1);
    axis_range(my - rr, my + rr, height, ts, &y0, &y1);
    for (int64_t yy = y0; yy <= y1; yy++)
      for (int64_t xx = x0; xx <= x1; xx++) {
        int64_t t = yy * tx_n + xx;
        if (lists) lists[cursor[t]++] = i;
        else counts[t]++;
        total++;
      }
  }
  free(cursor);
  free(order);
  return total;
}

/* Front-to-back blend of every tile (or of `tile_ids` only when n_sel >= 0):
 * _blend (gaussian_core.py:286-332) per pixel, background fill (354-355),
 * scatter (396-397).  Outputs: image (H*W*3), t_final (H*W), depth_img (H*W,
 * sum of w * z, not in the reference), touched (M, accumulated),
 * n_processed (T; the break index of _blend's loop, 324-325). */
void oracle_blend(int64_t m, const double* mean2d, const double* cov2d, const double* depth,
                  const double* radius, const double* color, const double* opac,
                  int64_t width, int64_t height, int64_t ts, const double* bg,
                  const int64_t* offsets, const int64_t* lists, int64_t n_sel,
                  const int64_t* tile_ids, double* image, double* t_final, double* depth_img,
                  int64_t* touched, int64_t* n_processed) {
  int64_t tx_n = (width + ts - 1) / ts, ty_n = (height + ts - 1) / ts;
  int64_t ntiles = tx_n * ty_n;
  int64_t nwork = n_sel >= 0 ? n_sel : ntiles;
  (void)m;
#pragma omp parallel
  {
    int64_t pmax = ts * ts;
    double* T = (double*)malloc(sizeof(double) * pmax);
    double* C = (double*)malloc(sizeof(double) * pmax * 3);
    double* D = (double*)malloc(sizeof(double) * pmax);
    double* px = (double*)malloc(sizeof(double) * pmax);
    double* py = (double*)malloc(sizeof(double) * pmax);
#pragma omp for schedule(dynamic, 1)
    for (int64_t w_i = 0; w_i < nwork; w_i++) {
      int64_t t = n_sel >= 0 ? tile_ids[w_i] : w_i;
      int64_t tyi = t / tx_n, txi = t % tx_n;
      int64_t tx = txi * ts, ty = tyi * ts;
      int64_t tw = ts < width - tx ? ts : width - tx, th = ts < height - ty ? ts : height - ty;
      int64_t np = tw * th;
      for (int64_t p = 0; p < np; p++) {
        T[p] = 1.0;
        C[3 * p] = C[3 * p + 1] = C[3 * p + 2] = 0.0;
        D[p] = 0.0;
        px[p] = (double)(tx + p % tw) + 0.5; /* _pixel_centers 335-337 */
        py[p] = (double)(ty + p / tw) + 0.5;
      }
      int64_t k0 = offsets[t], k1 = offsets[t + 1];
      int64_t processed = k1 - k0;
      for (int64_t k = k0; k < k1; k++) {
        int64_t s = lists[k];
        double a = cov2d[3 * s], b = cov2d[3 * s + 1], c = cov2d[3 * s + 2];
        double det = a * c - b * b;
        double ca = c / det, cb = -b / det, cc = a / det;
        double mx = mean2d[2 * s], my = mean2d[2 * s + 1];
        double r2 = radius[s] * radius[s];
        int64_t cnt = 0, any_active = 0;
        for (int64_t p = 0; p < np; p++) {
          double dx = px[p] - mx, dy = py[p] - my;
          double maha = (ca * (dx * dx) + ((2.0 * cb) * dx) * dy) + cc * (dy * dy);
          double sig = opac[s] * exp(-0.5 * maha);
          int inside = (dx * dx + dy * dy) <= r2;
          int active = T[p] >= TERM_EPS;
          sig = (inside && active) ? (sig > SIGMA_MAX ? SIGMA_MAX : sig) : 0.0;
          double w = T[p] * sig;
          C[3 * p + 0] = C[3 * p + 0] + w * color[3 * s + 0];
          C[3 * p + 1] = C[3 * p + 1] + w * color[3 * s + 1];
          C[3 * p + 2] = C[3 * p + 2] + w * color[3 * s + 2];
          D[p] = D[p] + w * depth[s];
          T[p] = T[p] * (1.0 - sig);
          cnt += w > 0.0;
          any_active |= T[p] >= TERM_EPS;
        }
        if (cnt) {
#pragma omp atomic
          touched[s] += cnt;
        }
        if (!any_active) {
          processed = k - k0 + 1;
          break;
        }
      }
      n_processed[t] = processed;
      for (int64_t p = 0; p < np; p++) {
        int64_t pix = (ty + p / tw) * width + (tx + p % tw);
        image[3 * pix + 0] = C[3 * p + 0] + T[p] * bg[0];
        image[3 * pix + 1] = C[3 * p + 1] + T[p] * bg[1];
        image[3 * pix + 2] = C[3 * p + 2] + T[p] * bg[2];
        t_final[pix] = T[p];
        depth_img[pix] = D[p];
      }
    }
    free(T);
    free(C);
    free(D);
    free(px);
    free(py);
  }
}

/* Robustness certificate: the smallest distance (px) between any splat's
 * bbox edge (mean -/+ radius) and the tile-boundary value it is compared
 * against.  If this exceeds the geometry's error bound (1 ulp of the
 * reference's sqrt), tile membership is provably identical to the reference. */
double oracle_margin(int64_t m, const double* mean2d, const double* radius, int64_t width,
                     int64_t height, int64_t ts) {
  double best = INFINITY;
  for (int64_t i = 0; i < m; i++) {
    double v[4] = {mean2d[2 * i] - radius[i], mean2d[2 * i] + radius[i],
                   mean2d[2 * i + 1] - radius[i], mean2d[2 * i + 1] + radius[i]};
    for (int e = 0; e < 4; e++) {
      int64_t size = e < 2 ? width : height;
      if (!(v[e] > -ts) || !(v[e] < size + ts)) continue;
      double q = v[e] / (double)ts;
      double near = round(q) * (double)ts;
      if (e % 2 == 0) { /* lo compared with min((j+1)ts, size) */
        double d = fabs(v[e] - near);
        double d2 = fabs(v[e] - (double)size);
        if (d2 < d) d = d2;
        if (d < best) best = d;
      } else {
        double d = fabs(v[e] - near);
        if (d < best) best = d;
      }
    }
  }
  return best;
}

int oracle_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

void oracle_set_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}
