/* TEST INFRASTRUCTURE ONLY — CPU parity oracle (see vf_oracle.h).
 *
 * Single-threaded plain-C restatement of the reference hot path.  Every
 * function cites the reference file:line it follows; paths are relative to
 * /root/reference/proj/.  Single-threaded on purpose: with one worker the
 * reference's racy last-writer-wins allocation requests become deterministic
 * (raster order, then DDA step) — SURVEY.md §8(a) A7.
 */
#define _POSIX_C_SOURCE 200809L
#include "vf_oracle.h"

#include <float.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

/* ------------------------------------------------------------------------ */
/* small math (include/voxfuse/core/types.hpp, pose.hpp, intrinsics.hpp)     */
/* ------------------------------------------------------------------------ */
typedef struct { double x, y, z; } d3;
typedef struct { float x, y, z; } f3;
typedef struct { float x, y, z, w; } f4;
typedef struct { int x, y, z; } i3;
typedef struct { double r[9]; double t[3]; } pose_t; /* p' = R p + t, R row-major */
typedef struct { double fx, fy, cx, cy; int width, height; } intr_t;

static d3 d3m(double x, double y, double z) { d3 v = {x, y, z}; return v; }
static d3 d3_add(d3 a, d3 b) { return d3m(a.x + b.x, a.y + b.y, a.z + b.z); }
static d3 d3_sub(d3 a, d3 b) { return d3m(a.x - b.x, a.y - b.y, a.z - b.z); }
static d3 d3_scale(d3 a, double s) { return d3m(a.x * s, a.y * s, a.z * s); }
static double d3_dot(d3 a, d3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
static double d3_norm(d3 a) { return sqrt(a.x * a.x + a.y * a.y + a.z * a.z); }
static d3 d3_cross(d3 a, d3 b) {
  return d3m(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}
static f3 f3m(float x, float y, float z) { f3 v = {x, y, z}; return v; }

/* Matrix3d * Vector3d, each row a left-to-right sum (pose.hpp:19). */
static d3 mat3_mul_vec(const double* r, d3 p) {
  return d3m(r[0] * p.x + r[1] * p.y + r[2] * p.z, r[3] * p.x + r[4] * p.y + r[5] * p.z,
             r[6] * p.x + r[7] * p.y + r[8] * p.z);
}
static void mat3_mul(const double* a, const double* b, double* out) {
  double o[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) o[i * 3 + j] = a[i * 3 + 0] * b[0 * 3 + j] + a[i * 3 + 1] * b[1 * 3 + j] + a[i * 3 + 2] * b[2 * 3 + j];
  memcpy(out, o, sizeof(o));
}
static void mat3_transpose(const double* a, double* out) {
  double o[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) o[j * 3 + i] = a[i * 3 + j];
  memcpy(out, o, sizeof(o));
}

static pose_t pose_identity(void) {
  pose_t p;
  memset(&p, 0, sizeof(p));
  p.r[0] = p.r[4] = p.r[8] = 1.0;
  return p;
}
static pose_t pose_from(const double* a) {
  pose_t p;
  memcpy(p.r, a, 9 * sizeof(double));
  memcpy(p.t, a + 9, 3 * sizeof(double));
  return p;
}
static void pose_to(const pose_t* p, double* a) {
  memcpy(a, p->r, 9 * sizeof(double));
  memcpy(a + 9, p->t, 3 * sizeof(double));
}
/* Pose::apply (pose.hpp:19): rotation * p + translation */
static d3 pose_apply(const pose_t* p, d3 v) {
  d3 q = mat3_mul_vec(p->r, v);
  return d3m(q.x + p->t[0], q.y + p->t[1], q.z + p->t[2]);
}
/* Pose::inverse (pose.hpp:30-33) */
static pose_t pose_inverse(const pose_t* p) {
  pose_t o;
  mat3_transpose(p->r, o.r);
  d3 t = mat3_mul_vec(o.r, d3m(p->t[0], p->t[1], p->t[2]));
  o.t[0] = -t.x;
  o.t[1] = -t.y;
  o.t[2] = -t.z;
  return o;
}
/* Pose::operator* (pose.hpp:26-28) */
static pose_t pose_compose(const pose_t* a, const pose_t* b) {
  pose_t o;
  mat3_mul(a->r, b->r, o.r);
  d3 t = mat3_mul_vec(a->r, d3m(b->t[0], b->t[1], b->t[2]));
  o.t[0] = t.x + a->t[0];
  o.t[1] = t.y + a->t[1];
  o.t[2] = t.z + a->t[2];
  return o;
}

/* intrinsics.hpp:35-43 */
static void project(const intr_t* in, d3 p, double* u, double* v) {
  *u = in->fx * p.x / p.z + in->cx;
  *v = in->fy * p.y / p.z + in->cy;
}
/* intrinsics.hpp:22-31 */
static intr_t intr_half(const intr_t* in) {
  intr_t h;
  h.fx = in->fx * 0.5;
  h.fy = in->fy * 0.5;
  h.cx = (in->cx - 0.5) * 0.5;
  h.cy = (in->cy - 0.5) * 0.5;
  h.width = (in->width + 1) / 2;
  h.height = (in->height + 1) / 2;
  return h;
}

/* ------------------------------------------------------------------------ */
/* Eigen decompositions the reference calls (restated as in oracle/eigen_shim */
/* /Eigen/Dense so that the shim-built reference and this oracle agree).     */
/* ------------------------------------------------------------------------ */
typedef struct { double c, s; } rot_t;
static rot_t rot_transpose(rot_t j) { rot_t r = {j.c, -j.s}; return r; }
static rot_t rot_mul(rot_t a, rot_t b) {
  rot_t r = {a.c * b.c - a.s * b.s, a.c * b.s + a.s * b.c};
  return r;
}
#define WM(m, n, r, c) (m)[(r) + (c) * (n)]
static void rotate_rows(double* m, int n, int p, int q, rot_t j) {
  if (j.c == 1 && j.s == 0) return;
  for (int i = 0; i < n; ++i) {
    const double xi = WM(m, n, p, i), yi = WM(m, n, q, i);
    WM(m, n, p, i) = j.c * xi + j.s * yi;
    WM(m, n, q, i) = -j.s * xi + j.c * yi;
  }
}
static void rotate_cols(double* m, int n, int p, int q, rot_t jj) {
  const rot_t j = rot_transpose(jj);
  if (j.c == 1 && j.s == 0) return;
  for (int i = 0; i < n; ++i) {
    const double xi = WM(m, n, i, p), yi = WM(m, n, i, q);
    WM(m, n, i, p) = j.c * xi + j.s * yi;
    WM(m, n, i, q) = -j.s * xi + j.c * yi;
  }
}
static rot_t make_jacobi(double x, double y, double z) {
  rot_t r = {1, 0};
  const double deno = 2.0 * fabs(y);
  if (deno < DBL_MIN) return r;
  const double tau = (x - z) / deno;
  const double w = sqrt(tau * tau + 1.0);
  const double t = tau > 0 ? 1.0 / (tau + w) : 1.0 / (tau - w);
  const double sign_t = t > 0 ? 1.0 : -1.0;
  const double n = 1.0 / sqrt(t * t + 1.0);
  r.s = -sign_t * (y / fabs(y)) * fabs(t) * n;
  r.c = n;
  return r;
}
static void real_2x2_jacobi_svd(const double* mat, int n, int p, int q, rot_t* jl, rot_t* jr) {
  double m00 = WM(mat, n, p, p), m01 = WM(mat, n, p, q), m10 = WM(mat, n, q, p), m11 = WM(mat, n, q, q);
  rot_t rot1;
  const double t = m00 + m11;
  const double d = m10 - m01;
  if (fabs(d) < DBL_MIN) {
    rot1.s = 0;
    rot1.c = 1;
  } else {
    const double u = t / d;
    const double tmp = sqrt(1.0 + u * u);
    rot1.s = 1.0 / tmp;
    rot1.c = u / tmp;
  }
  const double n00 = rot1.c * m00 + rot1.s * m10, n01 = rot1.c * m01 + rot1.s * m11;
  const double n11 = -rot1.s * m01 + rot1.c * m11;
  *jr = make_jacobi(n00, n01, n11);
  *jl = rot_mul(rot1, rot_transpose(*jr));
}
/* JacobiSVD of an n x n (n <= 6) column-major matrix: singular values sorted
 * descending, optional U and V. */
static void jacobi_svd(const double* in, int n, double* sv, double* u, double* v) {
  double w[36], uu[36], vv[36];
  double scale = 0;
  for (int i = 0; i < n * n; ++i) scale = fmax(scale, fabs(in[i]));
  if (!(scale > 0) || !isfinite(scale)) scale = 1.0;
  for (int i = 0; i < n * n; ++i) {
    w[i] = in[i] / scale;
    uu[i] = 0;
    vv[i] = 0;
  }
  for (int i = 0; i < n; ++i) WM(uu, n, i, i) = WM(vv, n, i, i) = 1.0;
  const double precision = 2.0 * DBL_EPSILON;
  double max_diag = 0;
  for (int i = 0; i < n; ++i) max_diag = fmax(max_diag, fabs(WM(w, n, i, i)));
  int finished = 0;
  while (!finished) {
    finished = 1;
    for (int p = 1; p < n; ++p) {
      for (int q = 0; q < p; ++q) {
        const double threshold = fmax(DBL_MIN, precision * max_diag);
        if (fabs(WM(w, n, p, q)) > threshold || fabs(WM(w, n, q, p)) > threshold) {
          finished = 0;
          rot_t jl, jr;
          real_2x2_jacobi_svd(w, n, p, q, &jl, &jr);
          rotate_rows(w, n, p, q, jl);
          rotate_cols(uu, n, p, q, rot_transpose(jl));
          rotate_cols(w, n, p, q, jr);
          rotate_cols(vv, n, p, q, jr);
          max_diag = fmax(max_diag, fmax(fabs(WM(w, n, p, p)), fabs(WM(w, n, q, q))));
        }
      }
    }
  }
  for (int i = 0; i < n; ++i) {
    const double a = WM(w, n, i, i);
    sv[i] = fabs(a);
    if (a < 0)
      for (int r = 0; r < n; ++r) WM(uu, n, r, i) = -WM(uu, n, r, i);
  }
  for (int i = 0; i < n; ++i) sv[i] *= scale;
  for (int i = 0; i < n; ++i) {
    int pos = i;
    for (int k = i + 1; k < n; ++k)
      if (sv[k] > sv[pos]) pos = k;
    if (sv[pos] == 0.0) break;
    if (pos != i) {
      double t = sv[i];
      sv[i] = sv[pos];
      sv[pos] = t;
      for (int r = 0; r < n; ++r) {
        t = WM(uu, n, r, i); WM(uu, n, r, i) = WM(uu, n, r, pos); WM(uu, n, r, pos) = t;
        t = WM(vv, n, r, i); WM(vv, n, r, i) = WM(vv, n, r, pos); WM(vv, n, r, pos) = t;
      }
    }
  }
  if (u) memcpy(u, uu, sizeof(double) * (size_t)(n * n));
  if (v) memcpy(v, vv, sizeof(double) * (size_t)(n * n));
}

/* LDLT with symmetric diagonal pivoting, then solve (Eigen LDLT; depth_tracker.hpp:209,214). */
static void ldlt_solve(const double* a_rowmajor, int n, const double* b, double* x) {
  double m[36];
  int trans[6];
  for (int r = 0; r < n; ++r)
    for (int c = 0; c < n; ++c) WM(m, n, r, c) = a_rowmajor[r * n + c];
  int zero = 0;
  double temp[6];
  for (int k = 0; k < n; ++k) trans[k] = k;
  for (int k = 0; k < n; ++k) {
    int big = k;
    double bigv = fabs(WM(m, n, k, k));
    for (int i = k + 1; i < n; ++i)
      if (fabs(WM(m, n, i, i)) > bigv) {
        bigv = fabs(WM(m, n, i, i));
        big = i;
      }
    trans[k] = big;
    if (k != big) {
      for (int c = 0; c < n; ++c) { double t = WM(m, n, k, c); WM(m, n, k, c) = WM(m, n, big, c); WM(m, n, big, c) = t; }
      for (int r = 0; r < n; ++r) { double t = WM(m, n, r, k); WM(m, n, r, k) = WM(m, n, r, big); WM(m, n, r, big) = t; }
    }
    const int rs = n - k - 1;
    if (k > 0) {
      for (int i = 0; i < k; ++i) temp[i] = WM(m, n, i, i) * WM(m, n, k, i);
      double s = 0;
      for (int i = 0; i < k; ++i) s = (i == 0) ? WM(m, n, k, 0) * temp[0] : s + WM(m, n, k, i) * temp[i];
      WM(m, n, k, k) -= s;
      for (int r = k + 1; r < n; ++r) {
        double t = 0;
        for (int i = 0; i < k; ++i) t = (i == 0) ? WM(m, n, r, 0) * temp[0] : t + WM(m, n, r, i) * temp[i];
        WM(m, n, r, k) -= t;
      }
    }
    const double akk = WM(m, n, k, k);
    const int pivot_ok = fabs(akk) > 0;
    if (k == 0 && !pivot_ok) {
      for (int j = 0; j < n; ++j) trans[j] = j;
      zero = 1;
      break;
    }
    if (rs > 0 && pivot_ok)
      for (int r = k + 1; r < n; ++r) WM(m, n, r, k) /= akk;
  }
  for (int i = 0; i < n; ++i) x[i] = b[i];
  for (int k = 0; k < n; ++k) { double t = x[k]; x[k] = x[trans[k]]; x[trans[k]] = t; }
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < i; ++j) x[i] -= WM(m, n, i, j) * x[j];
  for (int i = 0; i < n; ++i) {
    if (!zero && fabs(WM(m, n, i, i)) > DBL_MIN)
      x[i] /= WM(m, n, i, i);
    else
      x[i] = 0;
  }
  for (int i = n - 1; i >= 0; --i)
    for (int j = i + 1; j < n; ++j) x[i] -= WM(m, n, j, i) * x[j];
  for (int k = n - 1; k >= 0; --k) { double t = x[k]; x[k] = x[trans[k]]; x[trans[k]] = t; }
}

/* orthonormalize (src/pose.cpp:9-18) */
static void orthonormalize(const double* m_rowmajor, double* out) {
  double cm[9], u[9], v[9], sv[3];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) WM(cm, 3, r, c) = m_rowmajor[r * 3 + c];
  jacobi_svd(cm, 3, sv, u, v);
  double ur[9], vtr[9], r[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      ur[i * 3 + j] = WM(u, 3, i, j);
      vtr[i * 3 + j] = WM(v, 3, j, i);
    }
  mat3_mul(ur, vtr, r);
  const double det = r[0] * (r[4] * r[8] - r[5] * r[7]) - r[3] * (r[1] * r[8] - r[2] * r[7]) +
                     r[6] * (r[1] * r[5] - r[2] * r[4]);
  if (det < 0) {
    double flip[9] = {1, 0, 0, 0, 1, 0, 0, 0, -1}, t[9];
    mat3_mul(ur, flip, t);
    mat3_mul(t, vtr, r);
  }
  memcpy(out, r, sizeof(r));
}
/* I + skew(w) (pose.hpp:48-52; pose.cpp:23) */
static void i_plus_skew(const double* w, double* m) {
  m[0] = 1.0 + 0; m[1] = 0 + -w[2]; m[2] = 0 + w[1];
  m[3] = 0 + w[2]; m[4] = 1.0 + 0; m[5] = 0 + -w[0];
  m[6] = 0 + -w[1]; m[7] = 0 + w[0]; m[8] = 1.0 + 0;
}
/* pose_increment (src/pose.cpp:20-25) */
static pose_t pose_increment(const pose_t* pose, const double* twist) {
  double m[9], rd[9];
  i_plus_skew(twist, m);
  orthonormalize(m, rd);
  pose_t o;
  mat3_mul(rd, pose->r, o.r);
  d3 t = mat3_mul_vec(rd, d3m(pose->t[0], pose->t[1], pose->t[2]));
  o.t[0] = t.x + twist[3];
  o.t[1] = t.y + twist[4];
  o.t[2] = t.z + twist[5];
  return o;
}
/* pose_rotate_increment (src/pose.cpp:27-30) */
static pose_t pose_rotate_increment(const pose_t* pose, const double* omega) {
  double m[9], rd[9];
  i_plus_skew(omega, m);
  orthonormalize(m, rd);
  pose_t o;
  mat3_mul(rd, pose->r, o.r);
  memcpy(o.t, pose->t, sizeof(o.t));
  return o;
}

/* ------------------------------------------------------------------------ */
/* voxels and the block hash (voxel/voxel.hpp, volume/hash_volume.hpp)      */
/* ------------------------------------------------------------------------ */
typedef struct {
  int16_t x, y, z, pad;
  int32_t offset;
  int32_t block_state;
} entry_t; /* HashEntry, 16 B (hash_volume.hpp:24-28) */

enum { kBlockSide = 8, kBlockVolume = 512, kEntrySwappedOut = -1, kEntryUnallocated = -2 };

/* sdf_value_to_float / sdf_float_to_value (voxel.hpp:11-19) */
static float sdf_to_float(int16_t v) { return (float)v / 32767.0f; }
static int16_t sdf_from_float(float f) {
  f = f < -1.0f ? -1.0f : (1.0f < f ? 1.0f : f);
  return (int16_t)(f * 32767.0f);
}

/* hash_block_pos (hash_volume.hpp:32-37) */
uint32_t vfo_hash_block_pos(int x, int y, int z, uint32_t mask) {
  return (((uint32_t)x * 73856093u) ^ ((uint32_t)y * 19349669u) ^ ((uint32_t)z * 83492791u)) & mask;
}

typedef struct {
  int* slots;
  int n, top;
} freestack_t; /* FreeStack (hash_volume.hpp:62-110) */

static void fs_init(freestack_t* s, int n) {
  s->slots = (int*)malloc(sizeof(int) * (size_t)n);
  for (int i = 0; i < n; ++i) s->slots[i] = i;
  s->n = n;
  s->top = n;
}
static int fs_pop(freestack_t* s) {
  const int t = s->top - 1;
  if (t < 0) return -1;
  s->top = t;
  return s->slots[t];
}
static void fs_push(freestack_t* s, int slot) { s->slots[s->top++] = slot; }

struct vfo_ctx {
  vfo_config cfg;
  int tracking;
  int has_color;
  int vsize; /* bytes per voxel: 4 (VoxelS) or 8 (VoxelSRgb) */
  int ordered, entry_count;
  uint32_t mask;
  entry_t* entries;
  uint8_t* voxels;
  freestack_t vba_free, excess_free;
  /* AllocationScratch (allocation.hpp:26-40) */
  uint8_t* request;
  int16_t* request_pos;
  uint8_t* visibility;
  uint8_t* swap_visibility;
  int* visible_list;
  int n_visible;
  /* RangeImage (raycast.hpp:23-53) */
  int frag_w, frag_h;
  float* ranges;
  /* TrackingState (tracking_state.hpp:26-33) */
  pose_t pose;
  pose_t render_pose;
  f4* points;
  f4* normals;
  int maps_valid;
  int frame;
  intr_t depth_intr, rgb_intr;
  pose_t rgb_to_depth;
  /* ICP trace */
  double* trace;
  long trace_rows, trace_cap;
  /* TrackingState::surface_points / surface_colors (tracking_state.hpp:30-31) */
  f3* surf_points;
  f3* surf_colors;
  long n_surface;
  /* GlobalCache (swap.hpp:45-91): per-entry states + a memory block store
   * (block_store.cpp:28-56) holding VoxelCodec payloads, NULL = no data */
  uint8_t* swap_state;
  uint8_t** store;
  int payload_bytes;
};

static uint8_t* vox_bytes(vfo_ctx* c, long slot, int lin) {
  return c->voxels + ((size_t)slot * kBlockVolume + (size_t)lin) * (size_t)c->vsize;
}

/* find_entry (hash_volume.hpp:161-176) */
static int find_entry(const vfo_ctx* c, i3 b) {
  const int h = (int)vfo_hash_block_pos(b.x, b.y, b.z, c->mask) * c->cfg.bucket_size;
  int off = 0;
  for (int k = 0; k < c->cfg.bucket_size; ++k) {
    const entry_t* e = &c->entries[h + k];
    off = e->offset - 1;
    if (e->x == b.x && e->y == b.y && e->z == b.z && e->block_state >= kEntrySwappedOut) return h + k;
  }
  while (off >= 0) {
    const int idx = c->ordered + off;
    const entry_t* e = &c->entries[idx];
    if (e->x == b.x && e->y == b.y && e->z == b.z && e->block_state >= kEntrySwappedOut) return idx;
    off = e->offset - 1;
  }
  return -1;
}

/* HashVolume::read (hash_volume.hpp:180-200): returns voxel byte pointer or NULL */
static const uint8_t* volume_read(vfo_ctx* c, i3 p) {
  const i3 b = {p.x >> 3, p.y >> 3, p.z >> 3};
  const int lin = (p.x & 7) + (p.y & 7) * kBlockSide + (p.z & 7) * kBlockSide * kBlockSide;
  const int h = (int)vfo_hash_block_pos(b.x, b.y, b.z, c->mask) * c->cfg.bucket_size;
  int off = 0;
  for (int k = 0; k < c->cfg.bucket_size; ++k) {
    const entry_t* e = &c->entries[h + k];
    off = e->offset - 1;
    if (e->x == b.x && e->y == b.y && e->z == b.z && e->block_state >= 0)
      return vox_bytes(c, e->block_state, lin);
  }
  while (off >= 0) {
    const entry_t* e = &c->entries[c->ordered + off];
    if (e->x == b.x && e->y == b.y && e->z == b.z && e->block_state >= 0)
      return vox_bytes(c, e->block_state, lin);
    off = e->offset - 1;
  }
  return NULL;
}

enum { INS_INSERTED, INS_EXISTING, INS_REATTACHED, INS_VBA_FULL, INS_EXCESS_FULL };
/* insert_block (hash_volume.hpp:215-258) */
static int insert_block(vfo_ctx* c, i3 b, int* entry_index) {
  const int existing = find_entry(c, b);
  *entry_index = -1;
  if (existing >= 0) {
    entry_t* e = &c->entries[existing];
    *entry_index = existing;
    if (e->block_state >= 0) return INS_EXISTING;
    const int slot = fs_pop(&c->vba_free);
    if (slot < 0) return INS_VBA_FULL;
    e->block_state = slot;
    return INS_REATTACHED;
  }
  const int h = (int)vfo_hash_block_pos(b.x, b.y, b.z, c->mask) * c->cfg.bucket_size;
  for (int k = 0; k < c->cfg.bucket_size; ++k) {
    entry_t* e = &c->entries[h + k];
    if (e->block_state == kEntryUnallocated) {
      const int slot = fs_pop(&c->vba_free);
      if (slot < 0) return INS_VBA_FULL;
      e->x = (int16_t)b.x;
      e->y = (int16_t)b.y;
      e->z = (int16_t)b.z;
      e->block_state = slot;
      *entry_index = h + k;
      return INS_INSERTED;
    }
  }
  int last = h + c->cfg.bucket_size - 1;
  while (c->entries[last].offset > 0) last = c->ordered + c->entries[last].offset - 1;
  const int ex = fs_pop(&c->excess_free);
  if (ex < 0) return INS_EXCESS_FULL;
  const int slot = fs_pop(&c->vba_free);
  if (slot < 0) {
    fs_push(&c->excess_free, ex);
    return INS_VBA_FULL;
  }
  const int idx = c->ordered + ex;
  entry_t* e = &c->entries[idx];
  e->x = (int16_t)b.x;
  e->y = (int16_t)b.y;
  e->z = (int16_t)b.z;
  e->offset = 0;
  e->block_state = slot;
  c->entries[last].offset = ex + 1;
  *entry_index = idx;
  return INS_INSERTED;
}

/* ------------------------------------------------------------------------ */
/* allocation (engine/allocation.hpp)                                        */
/* ------------------------------------------------------------------------ */
static void mark_cell(vfo_ctx* c, i3 b) {
  const int idx = find_entry(c, b);
  if (idx >= 0) {
    /* allocation.hpp:152-153 — visibility write, overwritten by build_visible_list */
    c->visibility[idx] = c->entries[idx].block_state >= 0 ? 1 : 2;
  } else {
    const size_t slot = (size_t)vfo_hash_block_pos(b.x, b.y, b.z, c->mask) * (size_t)c->cfg.bucket_size;
    c->request_pos[3 * slot] = (int16_t)b.x;
    c->request_pos[3 * slot + 1] = (int16_t)b.y;
    c->request_pos[3 * slot + 2] = (int16_t)b.z;
    c->request[slot] = 1;
  }
}

/* detail::dda_cells (allocation.hpp:60-96) */
static void dda_cells(vfo_ctx* c, d3 p0, d3 p1) {
  const double a0[3] = {p0.x, p0.y, p0.z}, a1[3] = {p1.x, p1.y, p1.z};
  int cell[3], end[3], step[3];
  double t_max[3], t_delta[3];
  for (int a = 0; a < 3; ++a) {
    cell[a] = (int)floor(a0[a]);
    end[a] = (int)floor(a1[a]);
  }
  mark_cell(c, (i3){cell[0], cell[1], cell[2]});
  const double d[3] = {a1[0] - a0[0], a1[1] - a0[1], a1[2] - a0[2]};
  for (int a = 0; a < 3; ++a) {
    if (d[a] > 0) {
      step[a] = 1;
      t_max[a] = (cell[a] + 1 - a0[a]) / d[a];
      t_delta[a] = 1.0 / d[a];
    } else if (d[a] < 0) {
      step[a] = -1;
      t_max[a] = (cell[a] - a0[a]) / d[a];
      t_delta[a] = -1.0 / d[a];
    } else {
      step[a] = 0;
      t_max[a] = INFINITY;
      t_delta[a] = INFINITY;
    }
  }
  const int max_steps = abs(end[0] - cell[0]) + abs(end[1] - cell[1]) + abs(end[2] - cell[2]) + 3;
  for (int i = 0; i < max_steps && (cell[0] != end[0] || cell[1] != end[1] || cell[2] != end[2]); ++i) {
    int axis = 0;
    if (t_max[1] < t_max[axis]) axis = 1;
    if (t_max[2] < t_max[axis]) axis = 2;
    if (t_max[axis] > 1.0) break;
    cell[axis] += step[axis];
    t_max[axis] += t_delta[axis];
    mark_cell(c, (i3){cell[0], cell[1], cell[2]});
  }
}

/* mark_blocks (allocation.hpp:137-168), one worker */
static void mark_blocks(vfo_ctx* c, const float* depth, const pose_t* world_to_cam) {
  const pose_t cam_to_world = pose_inverse(world_to_cam);
  const double inv_block = 1.0 / (double)(c->cfg.voxel_size * (float)kBlockSide);
  const intr_t* in = &c->depth_intr;
  for (int y = 0; y < in->height; ++y) {
    for (int x = 0; x < in->width; ++x) {
      const float d = depth[(size_t)y * in->width + x];
      if (d <= 0.0f) continue;
      const d3 dir = d3m((x - in->cx) / in->fx, (y - in->cy) / in->fy, 1.0);
      const double near_d = fmax(0.001, (double)d - (double)c->cfg.mu) ;
      /* std::max(0.001, v) returns v unless 0.001 > v; fmax differs only on NaN */
      const d3 p0 = d3_scale(pose_apply(&cam_to_world, d3_scale(dir, near_d)), inv_block);
      const d3 p1 = d3_scale(pose_apply(&cam_to_world, d3_scale(dir, (double)d + (double)c->cfg.mu)), inv_block);
      dda_cells(c, p0, p1);
    }
  }
}

/* perform_allocations (allocation.hpp:179-206) */
static vfo_alloc_stats perform_allocations(vfo_ctx* c) {
  vfo_alloc_stats st = {0, 0, 0, 0};
  for (int i = 0; i < c->entry_count; ++i) {
    if (!c->request[i]) continue;
    c->request[i] = 0;
    ++st.requested;
    int ei;
    const i3 b = {c->request_pos[3 * i], c->request_pos[3 * i + 1], c->request_pos[3 * i + 2]};
    switch (insert_block(c, b, &ei)) {
      case INS_INSERTED: ++st.allocated; c->visibility[ei] = 1; break;
      case INS_EXISTING:
      case INS_REATTACHED: c->visibility[ei] = 1; break;
      case INS_VBA_FULL: ++st.dropped_vba_full; break;
      case INS_EXCESS_FULL: ++st.dropped_excess_full; break;
    }
  }
  return st;
}

/* block corner in world units: (int * 8 + off) computed in int, times a float
 * voxel size in FP32, then widened (allocation.hpp:110-112; raycast.hpp:292-294) */
static d3 block_corner(i3 b, int corner, float vs) {
  return d3m((double)((float)(b.x * kBlockSide + ((corner & 1) ? kBlockSide : 0)) * vs),
             (double)((float)(b.y * kBlockSide + ((corner & 2) ? kBlockSide : 0)) * vs),
             (double)((float)(b.z * kBlockSide + ((corner & 4) ? kBlockSide : 0)) * vs));
}

/* detail::block_projects_into_view (allocation.hpp:101-130) */
static int block_projects_into_view(i3 b, const pose_t* w2c, const intr_t* in, float vs, float near_clip,
                                    float far_clip, int margin) {
  double zmin = INFINITY, zmax = -INFINITY, xmin = INFINITY, xmax = -INFINITY, ymin = INFINITY, ymax = -INFINITY;
  int any_behind = 0;
  for (int corner = 0; corner < 8; ++corner) {
    const d3 cam = pose_apply(w2c, block_corner(b, corner, vs));
    zmin = cam.z < zmin ? cam.z : zmin; /* std::min(zmin, z) == (z < zmin ? z : zmin) */
    zmax = zmax < cam.z ? cam.z : zmax;
    if (cam.z <= 1e-6) {
      any_behind = 1;
      continue;
    }
    double u, v;
    project(in, cam, &u, &v);
    xmin = u < xmin ? u : xmin;
    xmax = xmax < u ? u : xmax;
    ymin = v < ymin ? v : ymin;
    ymax = ymax < v ? v : ymax;
  }
  if (zmax <= (double)near_clip || zmin >= (double)far_clip) return 0;
  if (any_behind) return 1;
  return xmax >= -margin && xmin <= in->width - 1 + margin && ymax >= -margin && ymin <= in->height - 1 + margin;
}

/* build_visible_list (allocation.hpp:216-248) */
static void build_visible_list(vfo_ctx* c, const pose_t* w2c) {
  for (int i = 0; i < c->entry_count; ++i) {
    const entry_t* e = &c->entries[i];
    if (e->block_state < kEntrySwappedOut) continue;
    const i3 b = {e->x, e->y, e->z};
    const int in_view = block_projects_into_view(b, w2c, &c->depth_intr, c->cfg.voxel_size, c->cfg.near_clip,
                                                 c->cfg.far_clip, c->cfg.margin_px);
    const int in_margin = in_view || block_projects_into_view(b, w2c, &c->depth_intr, c->cfg.voxel_size,
                                                              c->cfg.near_clip, c->cfg.far_clip, c->cfg.swap_margin_px);
    c->swap_visibility[i] = in_margin ? 1 : 0;
    c->visibility[i] = in_view ? (e->block_state >= 0 ? 1 : 2) : 0;
  }
  c->n_visible = 0;
  for (int i = 0; i < c->entry_count; ++i)
    if (c->visibility[i] == 1) c->visible_list[c->n_visible++] = i;
}

/* ------------------------------------------------------------------------ */
/* integration (engine/integration.hpp)                                      */
/* ------------------------------------------------------------------------ */
typedef struct {
  float r[9], t[3];
  float fx, fy, cx, cy;
  int width, height;
} camf_t; /* CameraF (integration.hpp:18-33) */

static camf_t camf(const pose_t* p, const intr_t* in) {
  camf_t c;
  for (int i = 0; i < 9; ++i) c.r[i] = (float)p->r[i];
  for (int i = 0; i < 3; ++i) c.t[i] = (float)p->t[i];
  c.fx = (float)in->fx;
  c.fy = (float)in->fy;
  c.cx = (float)in->cx;
  c.cy = (float)in->cy;
  c.width = in->width;
  c.height = in->height;
  return c;
}
static f3 camf_apply(const camf_t* c, f3 p) {
  return f3m(c->r[0] * p.x + c->r[1] * p.y + c->r[2] * p.z + c->t[0],
             c->r[3] * p.x + c->r[4] * p.y + c->r[5] * p.z + c->t[1],
             c->r[6] * p.x + c->r[7] * p.y + c->r[8] * p.z + c->t[2]);
}

/* update_voxel_depth (integration.hpp:40-74) */
static float update_voxel_depth(uint8_t* vox, f3 pt_model, const camf_t* cam, float mu, int max_weight,
                                const float* depth) {
  const f3 pc = camf_apply(cam, pt_model);
  if (pc.z <= 0) return -1;
  const float px = cam->fx * pc.x / pc.z + cam->cx;
  const float py = cam->fy * pc.y / pc.z + cam->cy;
  if (px < 1 || px > (float)cam->width - 2 || py < 1 || py > (float)cam->height - 2) return -1;
  const float dm = depth[(size_t)(int)(px + 0.5f) + (size_t)(int)(py + 0.5f) * (size_t)cam->width];
  if (dm <= 0.0f) return -1;
  const float eta = dm - pc.z;
  if (eta < -mu) return eta;
  int16_t sdf;
  memcpy(&sdf, vox, 2);
  const float old_f = sdf_to_float(sdf);
  const int old_w = vox[2];
  float new_f = fminf(1.0f, eta / mu); /* std::min(1.0f, x): x < 1 ? x : 1 — same for non-NaN */
  if (!(eta / mu < 1.0f)) new_f = 1.0f;
  int new_w = 1;
  new_f = (float)old_w * old_f + (float)new_w * new_f;
  new_w = old_w + new_w;
  new_f /= (float)new_w;
  new_w = new_w < max_weight ? new_w : max_weight;
  sdf = sdf_from_float(new_f);
  memcpy(vox, &sdf, 2);
  vox[2] = (uint8_t)new_w;
  return eta;
}

/* update_voxel_color (integration.hpp:78-101) */
static void update_voxel_color(uint8_t* vox, f3 pt_model, const camf_t* cam, int max_weight, const uint8_t* rgb) {
  const f3 pc = camf_apply(cam, pt_model);
  if (pc.z <= 0) return;
  const float px = cam->fx * pc.x / pc.z + cam->cx;
  const float py = cam->fy * pc.y / pc.z + cam->cy;
  if (px < 1 || px > (float)cam->width - 2 || py < 1 || py > (float)cam->height - 2) return;
  const uint8_t* s = rgb + 3 * ((size_t)(int)(px + 0.5f) + (size_t)(int)(py + 0.5f) * (size_t)cam->width);
  const int old_w = vox[6];
  const int new_w = old_w + 1 < max_weight ? old_w + 1 : max_weight;
  for (int ch = 0; ch < 3; ++ch) {
    const float b = ((float)vox[3 + ch] * (float)old_w + (float)s[ch]) / (float)(old_w + 1);
    vox[3 + ch] = (uint8_t)b;
  }
  vox[6] = (uint8_t)new_w;
}

/* integrate_frame, hash overload (integration.hpp:123-148) */
static void integrate_frame(vfo_ctx* c, const float* depth, const uint8_t* rgb, const pose_t* w2c) {
  const camf_t dcam = camf(w2c, &c->depth_intr);
  const int with_color = c->has_color && rgb != NULL;
  const pose_t d2r = pose_inverse(&c->rgb_to_depth);
  const pose_t rgbp = pose_compose(&d2r, w2c);
  const camf_t rcam = camf(&rgbp, &c->rgb_intr);
  const float vs = c->cfg.voxel_size, mu = c->cfg.mu;
  for (int li = 0; li < c->n_visible; ++li) {
    const entry_t* e = &c->entries[c->visible_list[li]];
    if (e->block_state < 0) continue;
    const float bx = (float)(e->x * kBlockSide), by = (float)(e->y * kBlockSide), bz = (float)(e->z * kBlockSide);
    for (int z = 0; z < kBlockSide; ++z)
      for (int y = 0; y < kBlockSide; ++y)
        for (int x = 0; x < kBlockSide; ++x) {
          const f3 pt = f3m((bx + ((float)x + 0.5f)) * vs, (by + ((float)y + 0.5f)) * vs, (bz + ((float)z + 0.5f)) * vs);
          uint8_t* vox = vox_bytes(c, e->block_state, x + y * kBlockSide + z * kBlockSide * kBlockSide);
          /* detail::integrate_voxel (integration.hpp:105-116) */
          if (c->cfg.stop_integrating_at_max && vox[2] >= c->cfg.max_weight) continue;
          const float eta = update_voxel_depth(vox, pt, &dcam, mu, c->cfg.max_weight, depth);
          if (with_color && fabsf(eta) <= mu) update_voxel_color(vox, pt, &rcam, c->cfg.max_weight, rgb);
        }
  }
}

/* ------------------------------------------------------------------------ */
/* raycast (engine/raycast.hpp)                                              */
/* ------------------------------------------------------------------------ */
/* create_expected_depths, hash overload (raycast.hpp:268-363) */
static void create_expected_depths(vfo_ctx* c, const pose_t* w2c) {
  const intr_t* in = &c->depth_intr;
  const int nf = c->frag_w * c->frag_h;
  for (int f = 0; f < nf; ++f) {
    c->ranges[2 * f] = FLT_MAX;
    c->ranges[2 * f + 1] = 0.0f;
  }
  const double near_clip = c->cfg.near_clip, far_clip = c->cfg.far_clip;
  for (int i = 0; i < c->n_visible; ++i) {
    const entry_t* e = &c->entries[c->visible_list[i]];
    const i3 bp = {e->x, e->y, e->z};
    double zmin = INFINITY, zmax = -INFINITY, xmin = INFINITY, xmax = -INFINITY, ymin = INFINITY, ymax = -INFINITY;
    int behind = 0;
    for (int corner = 0; corner < 8; ++corner) {
      const d3 cam = pose_apply(w2c, block_corner(bp, corner, c->cfg.voxel_size));
      zmin = cam.z < zmin ? cam.z : zmin;
      zmax = zmax < cam.z ? cam.z : zmax;
      if (cam.z <= 1e-6) {
        behind = 1;
        continue;
      }
      double u, v;
      project(in, cam, &u, &v);
      xmin = u < xmin ? u : xmin;
      xmax = xmax < u ? u : xmax;
      ymin = v < ymin ? v : ymin;
      ymax = ymax < v ? v : ymax;
    }
    if (behind || !(zmax > near_clip && zmin < far_clip)) continue;
    int px0 = (int)floor(xmin);
    px0 = px0 < 0 ? 0 : px0;
    int px1 = (int)ceil(xmax);
    px1 = in->width - 1 < px1 ? in->width - 1 : px1;
    int py0 = (int)floor(ymin);
    py0 = py0 < 0 ? 0 : py0;
    int py1 = (int)ceil(ymax);
    py1 = in->height - 1 < py1 ? in->height - 1 : py1;
    if (!(px0 <= px1 && py0 <= py1)) continue;
    const int fx0 = px0 / 16, fx1 = px1 / 16, fy0 = py0 / 16, fy1 = py1 / 16;
    const float fzmin = (float)(zmin < near_clip ? near_clip : zmin);
    const float fzmax = (float)(far_clip < zmax ? far_clip : zmax);
    for (int fy = fy0; fy <= fy1; ++fy)
      for (int fx = fx0; fx <= fx1; ++fx) {
        float* r = &c->ranges[2 * (fy * c->frag_w + fx)];
        r[0] = fzmin < r[0] ? fzmin : r[0];
        r[1] = r[1] < fzmax ? fzmax : r[1];
      }
  }
}

/* instrumentation (test infra): sample / probe counters of the last raycast */
static long g_ray_samples, g_ray_reads, g_ray_trilinear, g_ray_rays, g_ray_coarse;
long vfo_raycast_counters(long* out) {
  out[0] = g_ray_rays; out[1] = g_ray_samples; out[2] = g_ray_reads; out[3] = g_ray_trilinear; out[4] = g_ray_coarse;
  return 5;
}

/* HashSdfSampler::read (raycast.hpp:73-76) */
static int sdf_read(vfo_ctx* c, i3 v, float* value) {
  ++g_ray_reads;
  const uint8_t* vox = volume_read(c, v);
  int16_t sdf = 32767;
  int w = 0;
  if (vox) {
    memcpy(&sdf, vox, 2);
    w = vox[2];
  }
  *value = sdf_to_float(sdf);
  return vox != NULL && w > 0;
}

/* trilinear_sdf (raycast.hpp:102-117) */
static int trilinear_sdf(vfo_ctx* c, f3 p, float* out) {
  ++g_ray_trilinear;
  const f3 q = f3m(p.x - 0.5f, p.y - 0.5f, p.z - 0.5f);
  const i3 base = {(int)floorf(q.x), (int)floorf(q.y), (int)floorf(q.z)};
  const f3 f = f3m(q.x - (float)base.x, q.y - (float)base.y, q.z - (float)base.z);
  float value = 0.0f;
  for (int corner = 0; corner < 8; ++corner) {
    const int dx = corner & 1, dy = (corner >> 1) & 1, dz = (corner >> 2) & 1;
    float v;
    if (!sdf_read(c, (i3){base.x + dx, base.y + dy, base.z + dz}, &v)) {
      *out = 1.0f;
      return 0;
    }
    const float w = (dx ? f.x : 1 - f.x) * (dy ? f.y : 1 - f.y) * (dz ? f.z : 1 - f.z);
    value += w * v;
  }
  *out = value;
  return 1;
}

/* sdf_surface_normal (raycast.hpp:147-162) */
static int sdf_surface_normal(vfo_ctx* c, f3 p, f3* n) {
  float g[3];
  const float pa[3] = {p.x, p.y, p.z};
  for (int a = 0; a < 3; ++a) {
    float lo[3] = {pa[0], pa[1], pa[2]}, hi[3] = {pa[0], pa[1], pa[2]};
    lo[a] -= 1.0f;
    hi[a] += 1.0f;
    float vlo, vhi;
    const int ok_lo = trilinear_sdf(c, f3m(lo[0], lo[1], lo[2]), &vlo);
    const int ok_hi = trilinear_sdf(c, f3m(hi[0], hi[1], hi[2]), &vhi);
    if (!ok_lo || !ok_hi) return 0;
    g[a] = vhi - vlo;
  }
  const float len = sqrtf(g[0] * g[0] + g[1] * g[1] + g[2] * g[2]);
  if (len < 1e-12f) return 0;
  *n = f3m(g[0] / len, g[1] / len, g[2] / len);
  return 1;
}

/* cast_ray (raycast.hpp:171-263) */
static int cast_ray(vfo_ctx* c, int x, int y, const float* range, const pose_t* w2c, f3* hit_world) {
  if (!(range[0] <= range[1])) return 0;
  const intr_t* in = &c->depth_intr;
  const pose_t c2w = pose_inverse(w2c);
  const double inv_vox = 1.0 / (double)c->cfg.voxel_size;
  const d3 dir_cam = d3m((x - in->cx) / in->fx, (y - in->cy) / in->fy, 1.0);
  const d3 s0 = d3_scale(pose_apply(&c2w, d3_scale(dir_cam, (double)range[0])), inv_vox);
  const d3 e0 = d3_scale(pose_apply(&c2w, d3_scale(dir_cam, (double)range[1])), inv_vox);
  const f3 start = f3m((float)s0.x, (float)s0.y, (float)s0.z);
  const f3 end = f3m((float)e0.x, (float)e0.y, (float)e0.z);
  f3 dir = f3m(end.x - start.x, end.y - start.y, end.z - start.z);
  const float total = sqrtf(dir.x * dir.x + dir.y * dir.y + dir.z * dir.z);
  if (!(total > 0)) return 0;
  dir = f3m(dir.x / total, dir.y / total, dir.z / total);
  const float mu_vox = c->cfg.mu / c->cfg.voxel_size;
  const float fine_step = (8.0f < mu_vox) ? 8.0f : mu_vox; /* std::min(mu_vox, 8.f) */
  enum { COARSE, FINE, SURFACE } state = COARSE;
  float t = 0.0f, t_front = -1.0f, sdf_front = 1.0f;
  while (t <= total) {
    ++g_ray_samples;
    if (state == COARSE) ++g_ray_coarse;
    const f3 p = f3m(start.x + dir.x * t, start.y + dir.y * t, start.z + dir.z * t);
    float value;
    const int found = sdf_read(c, (i3){(int)floorf(p.x), (int)floorf(p.y), (int)floorf(p.z)}, &value);
    if (state == COARSE) {
      if (!found) {
        t += 8;
        continue;
      }
      state = FINE;
      t = 0.0f < t - 8 ? t - 8 : 0.0f; /* std::max(0.0f, t - 8) */
      continue;
    }
    if (!found) {
      if (state == SURFACE) state = FINE;
      t_front = -1.0f;
      t += fine_step;
      continue;
    }
    float sdf = value;
    if (state == FINE && sdf <= 0.0f) return 0; /* WRONG_SIDE */
    state = SURFACE;
    if (sdf <= 0.1f && sdf >= -0.5f) {
      float tri;
      if (trilinear_sdf(c, p, &tri)) sdf = tri;
    }
    if (sdf <= 0.0f) {
      if (t_front >= 0.0f && sdf_front > sdf && t - t_front <= 2.0f * mu_vox) {
        t = t + (t_front - t) * sdf / (sdf - sdf_front);
      } else {
        t += sdf * mu_vox;
      }
      float t_back = t, sdf_back = sdf;
      for (int i = 0; i < 2; ++i) {
        float tri;
        if (!trilinear_sdf(c, f3m(start.x + dir.x * t, start.y + dir.y * t, start.z + dir.z * t), &tri)) break;
        const float denom = sdf_back - tri;
        if (fabsf(denom) > 1e-12f && fabsf(t_back - t) > 1e-6f) {
          const float slope = denom / (t_back - t);
          t_back = t;
          sdf_back = tri;
          t -= tri / (fabsf(slope) > 1e-6f ? slope : 1.0f / mu_vox);
        } else {
          t += tri * mu_vox;
        }
      }
      const f3 h = f3m(start.x + dir.x * t, start.y + dir.y * t, start.z + dir.z * t);
      *hit_world = f3m(h.x * c->cfg.voxel_size, h.y * c->cfg.voxel_size, h.z * c->cfg.voxel_size);
      return 1;
    }
    t_front = t;
    sdf_front = sdf;
    {
      const float a = sdf * mu_vox;
      const float b = (a < 1.0f) ? 1.0f : a;     /* std::max(a, 1.0f) */
      t += (mu_vox < b) ? mu_vox : b;            /* std::min(b, mu_vox) */
    }
  }
  return 0;
}

/* render_maps (raycast.hpp:415-435) */
static void render_maps(vfo_ctx* c, const pose_t* w2c) {
  const intr_t* in = &c->depth_intr;
  g_ray_samples = g_ray_reads = g_ray_trilinear = g_ray_coarse = 0;
  g_ray_rays = (long)in->width * in->height;
  const size_t n = (size_t)in->width * (size_t)in->height;
  memset(c->points, 0, sizeof(f4) * n);
  memset(c->normals, 0, sizeof(f4) * n);
  for (int y = 0; y < in->height; ++y)
    for (int x = 0; x < in->width; ++x) {
      f3 hw;
      const float* range = &c->ranges[2 * ((y / 16) * c->frag_w + (x / 16))];
      if (!cast_ray(c, x, y, range, w2c, &hw)) continue;
      const f3 pv = f3m(hw.x / c->cfg.voxel_size, hw.y / c->cfg.voxel_size, hw.z / c->cfg.voxel_size);
      f3 nrm;
      if (!sdf_surface_normal(c, pv, &nrm)) continue;
      const size_t i = (size_t)y * in->width + x;
      c->points[i] = (f4){hw.x, hw.y, hw.z, 1.0f};
      c->normals[i] = (f4){nrm.x, nrm.y, nrm.z, 1.0f};
    }
}

/* sample_voxel_color (raycast.hpp:441-464) */
static f3 sample_voxel_color(vfo_ctx* c, f3 p) {
  if (!c->has_color) return f3m(0.0f, 0.0f, 0.0f);
  const f3 q = f3m(p.x - 0.5f, p.y - 0.5f, p.z - 0.5f);
  const i3 base = {(int)floorf(q.x), (int)floorf(q.y), (int)floorf(q.z)};
  const f3 f = f3m(q.x - (float)base.x, q.y - (float)base.y, q.z - (float)base.z);
  f3 sum = f3m(0.0f, 0.0f, 0.0f);
  float wsum = 0.0f;
  for (int corner = 0; corner < 8; ++corner) {
    const int dx = corner & 1, dy = (corner >> 1) & 1, dz = (corner >> 2) & 1;
    const i3 v = {base.x + dx, base.y + dy, base.z + dz};
    const uint8_t* vox = volume_read(c, v);
    if (!vox || vox[6] == 0) continue;
    const float w = (dx ? f.x : 1 - f.x) * (dy ? f.y : 1 - f.y) * (dz ? f.z : 1 - f.z);
    sum = f3m(sum.x + (float)vox[3] * w, sum.y + (float)vox[4] * w, sum.z + (float)vox[5] * w);
    wsum += w;
  }
  return wsum > 0.0f ? f3m(sum.x / wsum, sum.y / wsum, sum.z / wsum) : f3m(0.0f, 0.0f, 0.0f);
}

/* forward_project_points (raycast.hpp:495-509) */
static void forward_project_points(vfo_ctx* c, int stride) {
  const intr_t* in = &c->depth_intr;
  const float vs = c->cfg.voxel_size;
  c->n_surface = 0;
  for (int y = 0; y < in->height; y += stride)
    for (int x = 0; x < in->width; x += stride) {
      const f4 p = c->points[(size_t)y * in->width + x];
      if (p.w == 0.0f) continue;
      const f3 col = sample_voxel_color(c, f3m(p.x / vs, p.y / vs, p.z / vs));
      c->surf_points[c->n_surface] = f3m(p.x, p.y, p.z);
      c->surf_colors[c->n_surface] = f3m(col.x / 255.0f, col.y / 255.0f, col.z / 255.0f);
      ++c->n_surface;
    }
}

static float clampf(float v, float lo, float hi) { return v < lo ? lo : (hi < v ? hi : v); } /* std::clamp */

/* render_image (raycast.hpp:466-490): color 0 shaded grey, 1 colour */
static void render_image(vfo_ctx* c, int color, uint8_t* out) {
  const intr_t* in = &c->depth_intr;
  const float ax = (float)c->pose.r[6], ay = (float)c->pose.r[7], az = (float)c->pose.r[8];
  const float vs = c->cfg.voxel_size;
  memset(out, 0, (size_t)in->width * in->height * 3);
  for (int y = 0; y < in->height; ++y)
    for (int x = 0; x < in->width; ++x) {
      const size_t i = (size_t)y * in->width + x;
      const f4 p = c->points[i];
      if (p.w == 0.0f) continue;
      const f4 n = c->normals[i];
      const float shade = fabsf(n.x * ax + n.y * ay + n.z * az);
      if (!color || !c->has_color) {
        const uint8_t g = (uint8_t)(clampf(shade, 0.0f, 1.0f) * 255.0f);
        out[3 * i] = out[3 * i + 1] = out[3 * i + 2] = g;
      } else {
        const f3 s = sample_voxel_color(c, f3m(p.x / vs, p.y / vs, p.z / vs));
        const f3 col = f3m(s.x * shade, s.y * shade, s.z * shade);
        out[3 * i + 0] = (uint8_t)clampf(col.x, 0.0f, 255.0f);
        out[3 * i + 1] = (uint8_t)clampf(col.y, 0.0f, 255.0f);
        out[3 * i + 2] = (uint8_t)clampf(col.z, 0.0f, 255.0f);
      }
    }
}

/* ------------------------------------------------------------------------ */
/* swap engine (engine/swap.hpp)                                             */
/* ------------------------------------------------------------------------ */
enum { SW_INACTIVE = 0, SW_NEEDS_IN = 1, SW_IN_TRANSFER = 2, SW_ACTIVE = 3, SW_NEEDS_OUT = 4 };

/* VoxelCodec encode / decode (voxel.hpp:124-155): the first 3 (VoxelS) or 7
 * (VoxelSRgb) bytes of the oracle's voxel layout are exactly the codec bytes */
static int codec_bytes(const vfo_ctx* c) { return c->has_color ? 7 : 3; }

/* fuse_voxels (swap.hpp:96-131) on voxel bytes: out = active fused with host */
static void fuse_voxel(vfo_ctx* c, const uint8_t* host, uint8_t* active) {
  const int max_weight = c->cfg.max_weight;
  uint8_t out[8];
  memcpy(out, active, (size_t)c->vsize);
  const int wh = host[2], wa = active[2];
  if (wh + wa > 0) {
    if (wa == 0) {
      out[0] = host[0];
      out[1] = host[1];
      out[2] = host[2];
    } else if (wh == 0) {
      /* keep active */
    } else {
      int16_t hs, as;
      memcpy(&hs, host, 2);
      memcpy(&as, active, 2);
      const float f = (sdf_to_float(hs) * (float)wh + sdf_to_float(as) * (float)wa) / (float)(wh + wa);
      const int16_t q = sdf_from_float(f);
      memcpy(out, &q, 2);
      out[2] = (uint8_t)(wh + wa < max_weight ? wh + wa : max_weight);
    }
  }
  if (c->has_color) {
    const int ch = host[6], ca = active[6];
    if (ca == 0) {
      out[3] = host[3], out[4] = host[4], out[5] = host[5], out[6] = host[6];
    } else if (ch == 0) {
      /* active colour kept */
    } else {
      for (int k = 0; k < 3; ++k) {
        const float v = ((float)host[3 + k] * (float)ch + (float)active[3 + k] * (float)ca) / (float)(ch + ca);
        out[3 + k] = (uint8_t)v;
      }
      out[6] = (uint8_t)(ch + ca < max_weight ? ch + ca : max_weight);
    }
  }
  memcpy(active, out, (size_t)c->vsize);
}

/* request_swap_ins (swap.hpp:136-149) */
static void request_swap_ins(vfo_ctx* c) {
  for (int i = 0; i < c->entry_count; ++i) {
    const int visible = c->swap_visibility[i] != 0;
    if (c->swap_state[i] == SW_NEEDS_IN && !visible) c->swap_state[i] = SW_INACTIVE;
    if (c->entries[i].block_state == kEntrySwappedOut && c->store[i] && visible) c->swap_state[i] = SW_NEEDS_IN;
  }
}

/* execute_swap_in (swap.hpp:151-198) */
static void execute_swap_in(vfo_ctx* c, vfo_stats* m) {
  const int cap = c->cfg.swap_buffer_blocks;
  int staged = 0;
  for (int i = 0; i < c->entry_count && staged < cap; ++i) {
    if (c->swap_state[i] != SW_NEEDS_IN) continue;
    entry_t* e = &c->entries[i];
    int slot = e->block_state;
    if (slot < 0) {
      slot = fs_pop(&c->vba_free);
      if (slot < 0) break; /* deferred, request stays queued */
      e->block_state = slot;
    }
    c->swap_state[i] = SW_IN_TRANSFER;
    /* secondary integration of the host block into the active one */
    const int cb = codec_bytes(c);
    for (int v = 0; v < kBlockVolume; ++v) {
      uint8_t host[8] = {0};
      memcpy(host, c->store[i] + (size_t)v * cb, (size_t)cb);
      fuse_voxel(c, host, vox_bytes(c, slot, v));
    }
    free(c->store[i]); /* store.clear */
    c->store[i] = NULL;
    c->swap_state[i] = SW_ACTIVE;
    ++m->swapped_in;
    m->bytes_in += (uint64_t)c->payload_bytes + 4;
    ++staged;
  }
}

/* request_swap_outs (swap.hpp:204-227) */
static void request_swap_outs(vfo_ctx* c) {
  for (int i = 0; i < c->entry_count; ++i) {
    if (c->entries[i].block_state < 0) continue;
    const int visible = c->swap_visibility[i] != 0;
    switch (c->swap_state[i]) {
      case SW_INACTIVE: c->swap_state[i] = visible ? SW_ACTIVE : SW_NEEDS_OUT; break;
      case SW_ACTIVE: if (!visible) c->swap_state[i] = SW_NEEDS_OUT; break;
      case SW_NEEDS_OUT: if (visible) c->swap_state[i] = SW_ACTIVE; break;
      default: break;
    }
  }
}

/* execute_swap_out (swap.hpp:233-251) */
static void execute_swap_out(vfo_ctx* c, vfo_stats* m) {
  const int cap = c->cfg.swap_buffer_blocks;
  const int cb = codec_bytes(c);
  int processed = 0;
  for (int i = 0; i < c->entry_count && processed < cap; ++i) {
    if (c->swap_state[i] != SW_NEEDS_OUT) continue;
    entry_t* e = &c->entries[i];
    if (!c->store[i]) c->store[i] = (uint8_t*)malloc((size_t)c->payload_bytes);
    for (int v = 0; v < kBlockVolume; ++v) {
      uint8_t* vb = vox_bytes(c, e->block_state, v);
      memcpy(c->store[i] + (size_t)v * cb, vb, (size_t)cb);
      memset(vb, 0, (size_t)c->vsize); /* TVoxel{}: sdf 32767, weights and colour 0 */
      vb[0] = 0xFF;
      vb[1] = 0x7F;
    }
    fs_push(&c->vba_free, e->block_state);
    e->block_state = kEntrySwappedOut;
    c->swap_state[i] = SW_INACTIVE;
    ++processed;
    ++m->swapped_out;
    m->bytes_out += (uint64_t)c->payload_bytes + 4;
  }
}

long vfo_swap_states(const vfo_ctx* c, uint8_t* out) {
  if (out) memcpy(out, c->swap_state, (size_t)c->entry_count);
  return c->entry_count;
}
int vfo_store_read(const vfo_ctx* c, int idx, uint8_t* payload) {
  if (idx < 0 || idx >= c->entry_count || !c->store[idx]) return 0;
  if (payload) memcpy(payload, c->store[idx], (size_t)c->payload_bytes);
  return 1;
}
long vfo_store_count(const vfo_ctx* c) {
  long n = 0;
  for (int i = 0; i < c->entry_count; ++i) n += c->store[i] != NULL;
  return n;
}

/* disparity_to_depth (io/calibration.hpp:45-60) over an image
 * (disparity_image_to_depth, engine/view.hpp:18-28) */
void vfo_disparity_to_depth(const uint16_t* disp, long n, double a, double b, double fx, float max_depth,
                            float* depth) {
  const float fa = (float)a, fb = (float)b, ffx = (float)fx;
  for (long i = 0; i < n; ++i) {
    const float denom = fa - (float)disp[i];
    if (denom <= 0.0f) {
      depth[i] = 0.0f;
      continue;
    }
    const float z = 8.0f * fb * ffx / denom;
    depth[i] = (z > 0.0f && z <= max_depth) ? z : 0.0f;
  }
}

/* Pipeline::colourize_depth (pipeline_impl.hpp:225-239) */
void vfo_colourize_depth(const float* depth, int w, int h, uint8_t* out) {
  const size_t n = (size_t)w * h;
  float dmax = 0.0f;
  for (size_t i = 0; i < n; ++i) dmax = (dmax < depth[i]) ? depth[i] : dmax; /* std::max */
  memset(out, 0, n * 3);
  if (dmax <= 0.0f) return;
  for (size_t i = 0; i < n; ++i) {
    const float d = depth[i];
    if (d <= 0.0f) continue;
    const float t = d / dmax;
    out[3 * i + 0] = (uint8_t)(255 * (1.0f - t));
    out[3 * i + 1] = (uint8_t)(255 * (1.0f - fabsf(2 * t - 1)));
    out[3 * i + 2] = (uint8_t)(255 * t);
  }
}

/* ------------------------------------------------------------------------ */
/* depth pyramid (engine/pyramid.hpp)                                        */
/* ------------------------------------------------------------------------ */
/* downsample_depth (pyramid.hpp:35-65) */
static void downsample_depth(const float* src, int sw, int sh, float* dst) {
  const int dw = (sw + 1) / 2, dh = (sh + 1) / 2;
  for (int y = 0; y < dh; ++y)
    for (int x = 0; x < dw; ++x) {
      float dmin = 0.0f;
      for (int dy = 0; dy < 2; ++dy)
        for (int dx = 0; dx < 2; ++dx) {
          const int sx = 2 * x + dx, sy = 2 * y + dy;
          if (sx >= sw || sy >= sh) continue;
          const float d = src[(size_t)sy * sw + sx];
          if (d > 0.0f && (dmin <= 0.0f || d < dmin)) dmin = d;
        }
      float out = 0.0f;
      if (dmin > 0.0f) {
        float sum = 0.0f;
        int n = 0;
        for (int dy = 0; dy < 2; ++dy)
          for (int dx = 0; dx < 2; ++dx) {
            const int sx = 2 * x + dx, sy = 2 * y + dy;
            if (sx >= sw || sy >= sh) continue;
            const float d = src[(size_t)sy * sw + sx];
            if (d <= 0.0f || d > dmin + 0.05f) continue;
            sum += d;
            ++n;
          }
        out = sum / (float)n;
      }
      dst[(size_t)y * dw + x] = out;
    }
}

void vfo_depth_pyramid(const float* depth, int w, int h, int levels, float* out) {
  memcpy(out, depth, sizeof(float) * (size_t)w * (size_t)h);
  const float* src = out;
  float* dst = out + (size_t)w * h;
  for (int l = 1; l < levels; ++l) {
    downsample_depth(src, w, h, dst);
    src = dst;
    w = (w + 1) / 2;
    h = (h + 1) / 2;
    dst += (size_t)w * h;
  }
}

/* ------------------------------------------------------------------------ */
/* ICP (engine/depth_tracker.hpp)                                            */
/* ------------------------------------------------------------------------ */
typedef struct {
  double h[21], g[6], cost;
  int64_t count;
} icp_acc_t; /* detail::IcpAccum (depth_tracker.hpp:59-97) */

static void acc_add(icp_acc_t* a, const double* j, double r) {
  int k = 0;
  for (int x = 0; x < 6; ++x) {
    for (int y = x; y < 6; ++y) a->h[k++] += j[x] * j[y];
    a->g[x] += j[x] * r;
  }
  a->cost += r * r;
  ++a->count;
}
static void acc_merge(icp_acc_t* a, const icp_acc_t* o) {
  for (int i = 0; i < 21; ++i) a->h[i] += o->h[i];
  for (int i = 0; i < 6; ++i) a->g[i] += o->g[i];
  a->cost += o->cost;
  a->count += o->count;
}

/* detail::sample_map_bilinear (depth_tracker.hpp:37-55) */
static int sample_map_bilinear(const f4* map, int w, int h, double x, double y, float max_spread, d3* out) {
  if (x < 0 || y < 0 || x > w - 1.001 || y > h - 1.001) return 0;
  const int ix = (int)x, iy = (int)y;
  const double fx = x - ix, fy = y - iy;
  const f4 a = map[(size_t)iy * w + ix], b = map[(size_t)iy * w + ix + 1];
  const f4 c = map[(size_t)(iy + 1) * w + ix], d = map[(size_t)(iy + 1) * w + ix + 1];
  if (a.w == 0.0f || b.w == 0.0f || c.w == 0.0f || d.w == 0.0f) return 0;
#define MINF(p, q) ((q) < (p) ? (q) : (p))
#define MAXF(p, q) ((p) < (q) ? (q) : (p))
  const float lox = MINF(MINF(MINF(a.x, b.x), c.x), d.x), hix = MAXF(MAXF(MAXF(a.x, b.x), c.x), d.x);
  const float loy = MINF(MINF(MINF(a.y, b.y), c.y), d.y), hiy = MAXF(MAXF(MAXF(a.y, b.y), c.y), d.y);
  const float loz = MINF(MINF(MINF(a.z, b.z), c.z), d.z), hiz = MAXF(MAXF(MAXF(a.z, b.z), c.z), d.z);
#undef MINF
#undef MAXF
  const float sx = hix - lox, sy = hiy - loy, sz = hiz - loz;
  if (sqrtf(sx * sx + sy * sy + sz * sz) > max_spread) return 0;
  const float w0 = (float)((1 - fx) * (1 - fy)), w1 = (float)(fx * (1 - fy));
  const float w2 = (float)((1 - fx) * fy), w3 = (float)(fx * fy);
  out->x = (double)(a.x * w0 + b.x * w1 + c.x * w2 + d.x * w3);
  out->y = (double)(a.y * w0 + b.y * w1 + c.y * w2 + d.y * w3);
  out->z = (double)(a.z * w0 + b.z * w1 + c.z * w2 + d.z * w3);
  return 1;
}

/* detail::well_conditioned (depth_tracker.hpp:99-104); h row-major n x n */
static int well_conditioned(const double* h, int n, double max_condition) {
  double cm[36], sv[6];
  for (int r = 0; r < n; ++r)
    for (int c = 0; c < n; ++c) WM(cm, n, r, c) = h[r * n + c];
  jacobi_svd(cm, n, sv, NULL, NULL);
  const double smin = sv[n - 1], smax = sv[0];
  return smin > 0 && smax / smin < max_condition;
}

#define TRACE_ROW 48
/* trace row: level, iter, 21 H, 6 g, cost, count, rotation_only, evaluation
 * camera-to-world pose (12), 4 unused */
static void trace_row(vfo_ctx* c, int level, int iter, const icp_acc_t* t, int rot_only, const pose_t* c2w) {
  if (c->trace_rows >= c->trace_cap) {
    c->trace_cap = c->trace_cap ? c->trace_cap * 2 : 128;
    c->trace = (double*)realloc(c->trace, sizeof(double) * TRACE_ROW * (size_t)c->trace_cap);
  }
  double* r = c->trace + TRACE_ROW * c->trace_rows++;
  memset(r, 0, sizeof(double) * TRACE_ROW);
  r[0] = level;
  r[1] = iter;
  memcpy(r + 2, t->h, sizeof(t->h));
  memcpy(r + 23, t->g, sizeof(t->g));
  r[29] = t->cost;
  r[30] = (double)t->count;
  r[31] = rot_only;
  memcpy(r + 32, c2w->r, sizeof(c2w->r));
  memcpy(r + 41, c2w->t, sizeof(c2w->t));
}

typedef struct {
  pose_t pose;
  int ok, iterations, valid_points;
  double final_cost;
} track_result_t;

/* icp_track (depth_tracker.hpp:115-239); pyramid levels back to back */
static track_result_t icp_track(vfo_ctx* c, const float* pyr, const intr_t* intrs, int levels,
                                const pose_t* initial) {
  track_result_t res;
  res.pose = initial ? *initial : c->pose; /* result.pose = initial ? *initial : state.pose */
  res.ok = 0;
  res.iterations = 0;
  res.valid_points = 0;
  res.final_cost = 0;
  c->trace_rows = 0;
  if (!c->maps_valid) return res;
  const pose_t render_pose = c->pose;
  const intr_t* map_intr = &intrs[0];
  pose_t cam_to_world = pose_inverse(&res.pose);
  int iterations_total = 0, any_level_solved = 0;
  size_t offs[8];
  offs[0] = 0;
  for (int l = 1; l < levels; ++l) offs[l] = offs[l - 1] + (size_t)intrs[l - 1].width * intrs[l - 1].height;
  for (int level = levels - 1; level >= 0; --level) {
    const int rotation_only = level >= levels - c->cfg.rotation_only_levels;
    const float* depth = pyr + offs[level];
    const intr_t* in = &intrs[level];
    double accepted_cost = INFINITY;
    pose_t accepted_pose = cam_to_world;
    double pending[6] = {0, 0, 0, 0, 0, 0};
    int halvings = 0;
    for (int iter = 0; iter < c->cfg.max_iterations; ++iter) {
      const d3 rot_centre = rotation_only ? d3m(cam_to_world.t[0], cam_to_world.t[1], cam_to_world.t[2]) : d3m(0, 0, 0);
      icp_acc_t total;
      memset(&total, 0, sizeof(total));
      for (int y0 = 0; y0 < in->height; y0 += 8) { /* parallel_chunks(0, h, 8): chunk order merge */
        icp_acc_t acc;
        memset(&acc, 0, sizeof(acc));
        const int y1 = y0 + 8 < in->height ? y0 + 8 : in->height;
        for (int y = y0; y < y1; ++y)
          for (int x = 0; x < in->width; ++x) {
            const float d = depth[(size_t)y * in->width + x];
            if (d <= 0.0f) continue;
            /* unproject (intrinsics.hpp:39-43) */
            const d3 p_cam = d3m((x - in->cx) / in->fx * d, (y - in->cy) / in->fy * d, (double)d);
            const d3 p_world = pose_apply(&cam_to_world, p_cam);
            const d3 q = pose_apply(&render_pose, p_world);
            if (q.z <= 0.0) continue;
            double u, v;
            project(map_intr, q, &u, &v);
            d3 mp, mn;
            if (!sample_map_bilinear(c->points, map_intr->width, map_intr->height, u, v, c->cfg.icp_dist_threshold, &mp)) continue;
            if (!sample_map_bilinear(c->normals, map_intr->width, map_intr->height, u, v, 1.0f, &mn)) continue;
            const double nlen = d3_norm(mn);
            if (nlen < 1e-6) continue;
            mn = d3m(mn.x / nlen, mn.y / nlen, mn.z / nlen);
            /* icp_point_to_plane_term (depth_tracker.hpp:20-27) */
            const double r = d3_dot(d3_sub(p_world, mp), mn);
            d3 jr = d3_cross(p_world, mn);
            if (fabs(r) > (double)c->cfg.icp_dist_threshold) continue;
            if (rotation_only) jr = d3_cross(d3_sub(p_world, rot_centre), mn);
            const double j[6] = {jr.x, jr.y, jr.z, mn.x, mn.y, mn.z};
            acc_add(&acc, j, r);
          }
        acc_merge(&total, &acc);
      }
      trace_row(c, level, iter, &total, rotation_only, &cam_to_world);
      if (total.count < c->cfg.min_valid_points) {
        res.valid_points = (int)total.count;
        break;
      }
      const double cost = total.cost / (double)total.count;
      if (cost > accepted_cost) {
        const double sq = pending[0] * pending[0] + pending[1] * pending[1] + pending[2] * pending[2] +
                          pending[3] * pending[3] + pending[4] * pending[4] + pending[5] * pending[5];
        if (halvings < 4 && sq > 0) {
          ++halvings;
          for (int i = 0; i < 6; ++i) pending[i] *= 0.5;
          cam_to_world = rotation_only ? pose_rotate_increment(&accepted_pose, pending)
                                       : pose_increment(&accepted_pose, pending);
          continue;
        }
        cam_to_world = accepted_pose;
        break;
      }
      accepted_cost = cost;
      accepted_pose = cam_to_world;
      halvings = 0;
      double H[36];
      {
        int k = 0;
        for (int a = 0; a < 6; ++a)
          for (int b = a; b < 6; ++b) {
            H[a * 6 + b] = total.h[k];
            H[b * 6 + a] = total.h[k];
            ++k;
          }
      }
      double twist[6] = {0, 0, 0, 0, 0, 0};
      if (rotation_only) {
        double h3[9], g3[3];
        for (int a = 0; a < 3; ++a) {
          for (int b = 0; b < 3; ++b) h3[a * 3 + b] = H[a * 6 + b];
          g3[a] = -total.g[a];
        }
        if (!well_conditioned(h3, 3, c->cfg.max_condition)) return res;
        ldlt_solve(h3, 3, g3, twist);
        cam_to_world = pose_rotate_increment(&cam_to_world, twist);
      } else {
        double g6[6];
        for (int a = 0; a < 6; ++a) g6[a] = -total.g[a];
        if (!well_conditioned(H, 6, c->cfg.max_condition)) return res;
        ldlt_solve(H, 6, g6, twist);
        cam_to_world = pose_increment(&cam_to_world, twist);
      }
      memcpy(pending, twist, sizeof(pending));
      ++iterations_total;
      any_level_solved = 1;
      res.final_cost = cost;
      res.valid_points = (int)total.count;
      const double tn = sqrt(twist[0] * twist[0] + twist[1] * twist[1] + twist[2] * twist[2] +
                             twist[3] * twist[3] + twist[4] * twist[4] + twist[5] * twist[5]);
      if (tn < (double)c->cfg.convergence_eps) {
        accepted_pose = cam_to_world;
        break;
      }
    }
  }
  if (!any_level_solved) return res;
  res.pose = pose_inverse(&cam_to_world);
  res.ok = 1;
  res.iterations = iterations_total;
  return res;
}

/* ------------------------------------------------------------------------ */
/* context + pipeline (engine/pipeline_impl.hpp)                             */
/* ------------------------------------------------------------------------ */
vfo_ctx* vfo_create(const vfo_config* cfg, int tracking) {
  if (cfg->bucket_count <= 0 || (cfg->bucket_count & (cfg->bucket_count - 1)) != 0) return NULL;
  vfo_ctx* c = (vfo_ctx*)calloc(1, sizeof(vfo_ctx));
  c->cfg = *cfg;
  c->tracking = tracking;
  c->has_color = cfg->voxel_type == 2;
  c->vsize = c->has_color ? 8 : 4;
  c->ordered = cfg->bucket_count * cfg->bucket_size;
  c->entry_count = c->ordered + cfg->excess_count;
  c->mask = (uint32_t)(cfg->bucket_count - 1);
  c->entries = (entry_t*)calloc((size_t)c->entry_count, sizeof(entry_t));
  for (int i = 0; i < c->entry_count; ++i) c->entries[i].block_state = kEntryUnallocated;
  const size_t nvox = (size_t)cfg->block_count * kBlockVolume;
  c->voxels = (uint8_t*)calloc(nvox, (size_t)c->vsize);
  for (size_t i = 0; i < nvox; ++i) { /* VoxelS{} : sdf 32767, w 0 (voxel.hpp:29-30) */
    const int16_t s = 32767;
    memcpy(c->voxels + i * (size_t)c->vsize, &s, 2);
  }
  fs_init(&c->excess_free, cfg->excess_count);
  fs_init(&c->vba_free, cfg->block_count);
  c->request = (uint8_t*)calloc((size_t)c->entry_count, 1);
  c->request_pos = (int16_t*)calloc((size_t)c->entry_count * 3, sizeof(int16_t));
  c->visibility = (uint8_t*)calloc((size_t)c->entry_count, 1);
  c->swap_visibility = (uint8_t*)calloc((size_t)c->entry_count, 1);
  c->visible_list = (int*)calloc((size_t)c->entry_count, sizeof(int));
  c->depth_intr = (intr_t){cfg->fx, cfg->fy, cfg->cx, cfg->cy, cfg->width, cfg->height};
  c->rgb_intr = (intr_t){cfg->rgb_fx, cfg->rgb_fy, cfg->rgb_cx, cfg->rgb_cy, cfg->rgb_width, cfg->rgb_height};
  c->rgb_to_depth = pose_from(cfg->rgb_to_depth);
  c->frag_w = (cfg->width + 15) / 16;
  c->frag_h = (cfg->height + 15) / 16;
  c->ranges = (float*)calloc((size_t)c->frag_w * c->frag_h * 2, sizeof(float));
  c->points = (f4*)calloc((size_t)cfg->width * cfg->height, sizeof(f4));
  c->normals = (f4*)calloc((size_t)cfg->width * cfg->height, sizeof(f4));
  c->surf_points = (f3*)calloc((size_t)((cfg->width + 3) / 4) * ((cfg->height + 3) / 4), sizeof(f3));
  c->surf_colors = (f3*)calloc((size_t)((cfg->width + 3) / 4) * ((cfg->height + 3) / 4), sizeof(f3));
  c->pose = pose_identity();
  c->render_pose = pose_identity();
  c->swap_state = (uint8_t*)calloc((size_t)c->entry_count, 1);
  c->store = (uint8_t**)calloc((size_t)c->entry_count, sizeof(uint8_t*));
  c->payload_bytes = (c->has_color ? 7 : 3) * kBlockVolume;
  return c;
}

void vfo_destroy(vfo_ctx* c) {
  if (!c) return;
  free(c->entries);
  free(c->voxels);
  free(c->excess_free.slots);
  free(c->vba_free.slots);
  free(c->request);
  free(c->request_pos);
  free(c->visibility);
  free(c->swap_visibility);
  free(c->visible_list);
  free(c->ranges);
  free(c->points);
  free(c->normals);
  free(c->trace);
  free(c->surf_points);
  free(c->surf_colors);
  if (c->store)
    for (int i = 0; i < c->entry_count; ++i) free(c->store[i]);
  free(c->store);
  free(c->swap_state);
  free(c);
}

static double now_ms(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec * 1e3 + (double)ts.tv_nsec * 1e-6;
}

int vfo_stage_allocate(vfo_ctx* c, const float* depth, const double* pose, vfo_alloc_stats* out) {
  const pose_t p = pose_from(pose);
  mark_blocks(c, depth, &p);
  const vfo_alloc_stats st = perform_allocations(c);
  build_visible_list(c, &p);
  if (out) *out = st;
  return 0;
}
int vfo_stage_integrate(vfo_ctx* c, const float* depth, const uint8_t* rgb, const double* pose) {
  const pose_t p = pose_from(pose);
  integrate_frame(c, depth, rgb, &p);
  return 0;
}
int vfo_stage_raycast(vfo_ctx* c, const double* pose) {
  const pose_t p = pose_from(pose);
  create_expected_depths(c, &p);
  render_maps(c, &p);
  c->maps_valid = 1;
  c->render_pose = p;
  c->pose = p;
  if (c->has_color) forward_project_points(c, 4); /* pipeline_impl.hpp:218-221 */
  return 0;
}
int vfo_stage_forward_project(vfo_ctx* c) {
  forward_project_points(c, 4);
  return 0;
}
long vfo_surface_points(const vfo_ctx* c, float* points, float* colors) {
  if (points) memcpy(points, c->surf_points, sizeof(f3) * (size_t)c->n_surface);
  if (colors) memcpy(colors, c->surf_colors, sizeof(f3) * (size_t)c->n_surface);
  return c->n_surface;
}
int vfo_render_image(vfo_ctx* c, int color, uint8_t* out) {
  if (!c->maps_valid) return -1;
  render_image(c, color, out);
  return 0;
}

static track_result_t run_tracker(vfo_ctx* c, const float* depth, const pose_t* initial) {
  const int levels = c->cfg.levels;
  intr_t intrs[8];
  intrs[0] = c->depth_intr;
  size_t total = (size_t)intrs[0].width * intrs[0].height;
  for (int l = 1; l < levels; ++l) {
    intrs[l] = intr_half(&intrs[l - 1]);
    total += (size_t)intrs[l].width * intrs[l].height;
  }
  float* pyr = (float*)malloc(sizeof(float) * total);
  vfo_depth_pyramid(depth, c->depth_intr.width, c->depth_intr.height, levels, pyr);
  const track_result_t r = icp_track(c, pyr, intrs, levels, initial);
  free(pyr);
  return r;
}

int vfo_stage_icp_init(vfo_ctx* c, const float* depth, const double* initial, double* out_pose, int* out_iters,
                       double* out_cost, int* out_valid) {
  pose_t init;
  if (initial) init = pose_from(initial);
  const track_result_t r = run_tracker(c, depth, initial ? &init : NULL);
  pose_to(&r.pose, out_pose);
  *out_iters = r.iterations;
  *out_cost = r.final_cost;
  *out_valid = r.valid_points;
  return r.ok;
}

int vfo_stage_icp(vfo_ctx* c, const float* depth, double* out_pose, int* out_iters, double* out_cost, int* out_valid) {
  const track_result_t r = run_tracker(c, depth, NULL);
  pose_to(&r.pose, out_pose);
  *out_iters = r.iterations;
  *out_cost = r.final_cost;
  *out_valid = r.valid_points;
  return r.ok;
}

int vfo_process(vfo_ctx* c, const float* depth, const uint8_t* rgb, const double* pose, vfo_stats* st) {
  const double t_start = now_ms();
  vfo_stats s;
  memset(&s, 0, sizeof(s));
  s.frame = c->frame;
  s.tracking_ok = 1;
  double t0 = now_ms();
  if (c->tracking) {
    if (c->frame > 0) { /* pipeline_impl.hpp:78-86 */
      const track_result_t r = run_tracker(c, depth, NULL);
      s.tracking_ok = r.ok;
      s.tracking_iterations = r.iterations;
      s.tracking_cost = r.final_cost;
      if (r.ok) c->pose = r.pose;
    }
  } else {
    if (!pose) return -1;
    c->pose = pose_from(pose);
  }
  s.ms_tracking = now_ms() - t0;
  t0 = now_ms();
  mark_blocks(c, depth, &c->pose);
  const vfo_alloc_stats a = perform_allocations(c);
  s.blocks_allocated = a.allocated;
  s.allocation_dropped = a.dropped_vba_full + a.dropped_excess_full;
  build_visible_list(c, &c->pose);
  s.visible_blocks = c->n_visible;
  s.ms_allocation = now_ms() - t0;
  t0 = now_ms();
  integrate_frame(c, depth, rgb, &c->pose);
  s.ms_integration = now_ms() - t0;
  t0 = now_ms();
  if (c->cfg.use_swapping) { /* pipeline_impl.hpp:104-113 */
    request_swap_ins(c);
    execute_swap_in(c, &s);
    request_swap_outs(c);
    execute_swap_out(c, &s);
  }
  s.ms_swapping = now_ms() - t0;
  t0 = now_ms();
  create_expected_depths(c, &c->pose);
  render_maps(c, &c->pose);
  c->maps_valid = 1;
  c->render_pose = c->pose;
  if (c->has_color) forward_project_points(c, 4); /* pipeline_impl.hpp:218-221 */
  s.ms_raycast = now_ms() - t0;
  pose_to(&c->pose, s.pose);
  s.ms_total = now_ms() - t_start;
  ++c->frame;
  if (st) *st = s;
  return 0;
}

void vfo_get_pose(const vfo_ctx* c, double* out) { pose_to(&c->pose, out); }
void vfo_set_pose(vfo_ctx* c, const double* pose) { c->pose = pose_from(pose); }
int vfo_get_maps(const vfo_ctx* c, float* points, float* normals) {
  if (!c->maps_valid) return -1;
  const size_t n = (size_t)c->cfg.width * c->cfg.height;
  memcpy(points, c->points, sizeof(f4) * n);
  memcpy(normals, c->normals, sizeof(f4) * n);
  return 0;
}
int vfo_set_maps(vfo_ctx* c, const float* points, const float* normals, const double* render_pose) {
  const size_t n = (size_t)c->cfg.width * c->cfg.height;
  memcpy(c->points, points, sizeof(f4) * n);
  memcpy(c->normals, normals, sizeof(f4) * n);
  c->pose = pose_from(render_pose);
  c->render_pose = c->pose;
  c->maps_valid = 1;
  return 0;
}
long vfo_export_entries(const vfo_ctx* c, void* out) {
  if (out) memcpy(out, c->entries, sizeof(entry_t) * (size_t)c->entry_count);
  return c->entry_count;
}
long vfo_export_voxels(const vfo_ctx* c, void* out) {
  const size_t n = (size_t)c->cfg.block_count * kBlockVolume * (size_t)c->vsize;
  if (out) memcpy(out, c->voxels, n);
  return (long)n;
}
long vfo_visible_list(const vfo_ctx* c, int* out) {
  if (out) memcpy(out, c->visible_list, sizeof(int) * (size_t)c->n_visible);
  return c->n_visible;
}
long vfo_export_ranges(const vfo_ctx* c, float* out) {
  const long n = (long)c->frag_w * c->frag_h;
  if (out) memcpy(out, c->ranges, sizeof(float) * 2 * (size_t)n);
  return n;
}
long vfo_allocated_blocks(const vfo_ctx* c) { return c->cfg.block_count - c->vba_free.top; }
void vfo_free_stacks(const vfo_ctx* c, int* vba_top, int* vba_slots, int* excess_top, int* excess_slots) {
  if (vba_top) *vba_top = c->vba_free.top;
  if (vba_slots) memcpy(vba_slots, c->vba_free.slots, sizeof(int) * (size_t)c->vba_free.n);
  if (excess_top) *excess_top = c->excess_free.top;
  if (excess_slots) memcpy(excess_slots, c->excess_free.slots, sizeof(int) * (size_t)c->excess_free.n);
}
long vfo_icp_trace(const vfo_ctx* c, double* out, long max_rows) {
  const long n = c->trace_rows < max_rows ? c->trace_rows : max_rows;
  if (out && n > 0) memcpy(out, c->trace, sizeof(double) * TRACE_ROW * (size_t)n);
  return c->trace_rows;
}

/* volume_digest: FNV-1a over allocated entries ascending, pos (6 B) then the
 * little-endian VoxelCodec bytes of each voxel (pipeline_impl.hpp:144-164,
 * voxel.hpp:123-155). */
uint64_t vfo_digest(const vfo_ctx* c) {
  uint64_t h = 1469598103934665603ull;
#define FNV(byte) do { h ^= (uint8_t)(byte); h *= 1099511628211ull; } while (0)
  for (int i = 0; i < c->entry_count; ++i) {
    const entry_t* e = &c->entries[i];
    if (e->block_state < 0) continue;
    const uint8_t* pb = (const uint8_t*)e;
    for (int k = 0; k < 6; ++k) FNV(pb[k]);
    for (int v = 0; v < kBlockVolume; ++v) {
      const uint8_t* vx = c->voxels + ((size_t)e->block_state * kBlockVolume + (size_t)v) * (size_t)c->vsize;
      FNV(vx[0]);
      FNV(vx[1]);
      FNV(vx[2]);
      if (c->has_color) {
        FNV(vx[3]);
        FNV(vx[4]);
        FNV(vx[5]);
        FNV(vx[6]);
      }
    }
  }
#undef FNV
  return h;
}

/* ------------------------------------------------------------------------ */
/* synthetic scene renderer (src/synthetic.cpp:19-108)                       */
/* ------------------------------------------------------------------------ */
typedef struct {
  double t;
  d3 point, normal;
  float albedo[3];
} hit_t;

static hit_t trace(int ns, const double* spheres, int np, const double* planes, d3 origin, d3 dir, double near_clip,
                   double far_clip) {
  hit_t best;
  best.t = INFINITY;
  best.point = best.normal = d3m(0, 0, 0);
  best.albedo[0] = best.albedo[1] = best.albedo[2] = 0;
  for (int i = 0; i < ns; ++i) {
    const double* s = spheres + 7 * i;
    const d3 centre = d3m(s[0], s[1], s[2]);
    const d3 oc = d3_sub(origin, centre);
    const double a = d3_dot(dir, dir);
    const double b = 2.0 * d3_dot(oc, dir);
    const double cc = d3_dot(oc, oc) - s[3] * s[3];
    const double disc = b * b - 4 * a * cc;
    if (disc < 0) continue;
    const double sq = sqrt(disc);
    const double ts[2] = {(-b - sq) / (2 * a), (-b + sq) / (2 * a)};
    for (int k = 0; k < 2; ++k) {
      const double t = ts[k];
      if (t > near_clip && t < far_clip && t < best.t) {
        best.t = t;
        best.point = d3_add(origin, d3_scale(dir, t));
        const d3 nn = d3_sub(best.point, centre);
        const double len = d3_norm(nn);
        best.normal = len > 0 ? d3m(nn.x / len, nn.y / len, nn.z / len) : nn;
        best.albedo[0] = (float)s[4];
        best.albedo[1] = (float)s[5];
        best.albedo[2] = (float)s[6];
      }
    }
  }
  for (int i = 0; i < np; ++i) {
    const double* p = planes + 9 * i;
    const d3 n = d3m(p[0], p[1], p[2]);
    const double denom = d3_dot(n, dir);
    if (fabs(denom) < 1e-12) continue;
    const double t = (p[3] - d3_dot(n, origin)) / denom;
    if (t > near_clip && t < far_clip && t < best.t) {
      best.t = t;
      best.point = d3_add(origin, d3_scale(dir, t));
      best.normal = denom < 0 ? n : d3m(-n.x, -n.y, -n.z);
      float alb[3] = {(float)p[4], (float)p[5], (float)p[6]};
      if (p[7] != 0.0) {
        const double na[3] = {fabs(n.x), fabs(n.y), fabs(n.z)};
        int drop = 0;
        if (na[1] > na[drop]) drop = 1;
        if (na[2] > na[drop]) drop = 2;
        const double pt[3] = {best.point.x, best.point.y, best.point.z};
        double uv[2] = {0, 0};
        int k = 0;
        for (int axis = 0; axis < 3; ++axis) {
          if (axis == drop) continue;
          uv[k++] = pt[axis];
        }
        const long pu = (long)floor(uv[0] / p[8]);
        const long pv = (long)floor(uv[1] / p[8]);
        if (((pu + pv) & 1) != 0)
          for (int ch = 0; ch < 3; ++ch) alb[ch] *= 0.35f;
      }
      memcpy(best.albedo, alb, sizeof(alb));
    }
  }
  return best;
}

void vfo_render_depth(int ns, const double* spheres, int np, const double* planes, const double* w2c, double fx,
                      double fy, double cx, double cy, int w, int h, double near_clip, double far_clip, float* out) {
  const pose_t p = pose_from(w2c);
  const pose_t c2w = pose_inverse(&p);
  const d3 origin = d3m(c2w.t[0], c2w.t[1], c2w.t[2]);
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x) {
      const d3 dir = mat3_mul_vec(c2w.r, d3m((x - cx) / fx, (y - cy) / fy, 1.0));
      const hit_t hit = trace(ns, spheres, np, planes, origin, dir, near_clip, far_clip);
      out[(size_t)y * w + x] = isfinite(hit.t) ? (float)hit.t : 0.0f;
    }
}

void vfo_render_rgb(int ns, const double* spheres, int np, const double* planes, const double* w2c, double fx,
                    double fy, double cx, double cy, int w, int h, double near_clip, double far_clip, uint8_t* out) {
  const pose_t p = pose_from(w2c);
  const pose_t c2w = pose_inverse(&p);
  const d3 origin = d3m(c2w.t[0], c2w.t[1], c2w.t[2]);
  d3 light = d3m(0.3, -0.7, -0.5);
  const double ll = d3_norm(light);
  light = d3m(light.x / ll, light.y / ll, light.z / ll);
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x) {
      const d3 dir = mat3_mul_vec(c2w.r, d3m((x - cx) / fx, (y - cy) / fy, 1.0));
      const hit_t hit = trace(ns, spheres, np, planes, origin, dir, near_clip, far_clip);
      uint8_t* o = out + 3 * ((size_t)y * w + x);
      if (!isfinite(hit.t)) {
        o[0] = o[1] = o[2] = 0;
        continue;
      }
      const double dd = d3_dot(hit.normal, d3m(-light.x, -light.y, -light.z));
      const float shade = 0.3f + 0.7f * (float)(0.0 < dd ? dd : 0.0);
      for (int ch = 0; ch < 3; ++ch) {
        const float cv = hit.albedo[ch] * shade * 255.0f;
        o[ch] = (uint8_t)(cv < 255.f ? cv : 255.f);
      }
    }
}
