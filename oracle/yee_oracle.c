/*
 * yee_oracle.c — CPU ORACLE (test infrastructure; see yee_oracle.h).
 * Build: oracle/Makefile, gcc -O3 -fopenmp -ffp-contract=off (the
 * reference's own build rule, proj/CMakeLists.txt:12-14).
 *
 * Every update keeps the reference operand order (kernels.hpp:10-25):
 *   difference first, then scale, then the signed combination, then the
 *   accumulation. Extended form: v = A*v + (C1*(a-b) - C2*(c-d)). With A = 1
 *   this is bit-identical to the reference's v += C1*(a-b) - C2*(c-d).
 */
#include "yee_oracle.h"

#include <stdlib.h>
#include <string.h>

#include "../include/yeeb200_inputs.h"

#define OMP_FOR _Pragma("omp parallel for schedule(static) num_threads(nthreads)")

/* staggering.hpp:34-39: node axes have extent n+1. */
void yo_comp_extents(int nx, int ny, int nz, int comp, int ext[3]) {
  const int n[3] = {nx, ny, nz};
  const int axis = comp % 3;
  const int electric = comp < 3;
  for (int a = 0; a < 3; ++a) {
    const int node = electric ? (a != axis) : (a == axis);
    ext[a] = n[a] + (node ? 1 : 0);
  }
}

int64_t yo_comp_size(int nx, int ny, int nz, int comp) {
  int e[3];
  yo_comp_extents(nx, ny, nz, comp, e);
  return (int64_t)e[0] * e[1] * e[2];
}

static inline int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

typedef struct {
  int nx, ny, nz;
  int e[6][3];
} geo;

static geo make_geo(const yo_state* s) {
  geo g;
  g.nx = s->nx;
  g.ny = s->ny;
  g.nz = s->nz;
  for (int c = 0; c < 6; ++c) yo_comp_extents(s->nx, s->ny, s->nz, c, g.e[c]);
  return g;
}

#define AT(c, i, j, k) (((int64_t)(k) * g.e[c][1] + (j)) * g.e[c][0] + (i))
/* Per-cell coefficient index of DoF (i,j,k): the cell clamped into the grid.
 * CROW is its (j,k) part, hoisted out of the i loops. */
#define CROW(j, k) (((int64_t)clampi(k, 0, g.nz - 1) * g.ny + clampi(j, 0, g.ny - 1)) * g.nx)
#define CELL(i, j, k) (CROW(j, k) + ((i) < g.nx ? (i) : g.nx - 1))

/* kernels.hpp:18-20 / :27-44, over curl_updatable_box (staggering.hpp:70-77). */
void yo_ampere(yo_state* s, const yo_coeffs* c, int nthreads) {
  const geo g = make_geo(s);
  float *ex = s->f[0], *ey = s->f[1], *ez = s->f[2];
  const float *hx = s->f[3], *hy = s->f[4], *hz = s->f[5];
  /* ex: i in [0,nx), j in [1,ny), k in [1,nz) */
  OMP_FOR
  for (int k = 1; k < g.nz; ++k)
    for (int j = 1; j < g.ny; ++j) {
      const int64_t crow = CROW(j, k);
      for (int i = 0; i < g.nx; ++i) {
        const int64_t cl = crow + (i < g.nx ? i : g.nx - 1);
        const float A = c->ca ? c->ca[cl] : c->ca_s;
        const float C1 = c->cb ? c->cb[cl] : c->cdy[j];
        const float C2 = c->cb ? c->cb[cl] : c->cdz[k];
        const int64_t p = AT(0, i, j, k);
        const float d1 = hz[AT(5, i, j, k)] - hz[AT(5, i, j - 1, k)];
        const float d2 = hy[AT(4, i, j, k)] - hy[AT(4, i, j, k - 1)];
        const float t1 = C1 * d1;
        const float t2 = C2 * d2;
        const float inc = t1 - t2;
        ex[p] = A * ex[p] + inc;
      }
    }
  /* ey: i in [1,nx), j in [0,ny), k in [1,nz) */
  OMP_FOR
  for (int k = 1; k < g.nz; ++k)
    for (int j = 0; j < g.ny; ++j) {
      const int64_t crow = CROW(j, k);
      for (int i = 1; i < g.nx; ++i) {
        const int64_t cl = crow + (i < g.nx ? i : g.nx - 1);
        const float A = c->ca ? c->ca[cl] : c->ca_s;
        const float C1 = c->cb ? c->cb[cl] : c->cdz[k];
        const float C2 = c->cb ? c->cb[cl] : c->cdx[i];
        const int64_t p = AT(1, i, j, k);
        const float d1 = hx[AT(3, i, j, k)] - hx[AT(3, i, j, k - 1)];
        const float d2 = hz[AT(5, i, j, k)] - hz[AT(5, i - 1, j, k)];
        const float t1 = C1 * d1;
        const float t2 = C2 * d2;
        const float inc = t1 - t2;
        ey[p] = A * ey[p] + inc;
      }
    }
  /* ez: i in [1,nx), j in [1,ny), k in [0,nz) */
  OMP_FOR
  for (int k = 0; k < g.nz; ++k)
    for (int j = 1; j < g.ny; ++j) {
      const int64_t crow = CROW(j, k);
      for (int i = 1; i < g.nx; ++i) {
        const int64_t cl = crow + (i < g.nx ? i : g.nx - 1);
        const float A = c->ca ? c->ca[cl] : c->ca_s;
        const float C1 = c->cb ? c->cb[cl] : c->cdx[i];
        const float C2 = c->cb ? c->cb[cl] : c->cdy[j];
        const int64_t p = AT(2, i, j, k);
        const float d1 = hy[AT(4, i, j, k)] - hy[AT(4, i - 1, j, k)];
        const float d2 = hx[AT(3, i, j, k)] - hx[AT(3, i, j - 1, k)];
        const float t1 = C1 * d1;
        const float t2 = C2 * d2;
        const float inc = t1 - t2;
        ez[p] = A * ez[p] + inc;
      }
    }
}

/* pec_boxes (staggering.hpp:81-86): every E DoF outside curl_updatable_box,
 * i.e. the node planes idx[ax] == 0 and idx[ax] == n[ax] of each axis ax
 * tangential to the component (the six outer faces; edges are visited
 * twice, writing the same +0). */
void yo_pec(yo_state* s) {
  const geo g = make_geo(s);
  const int n[3] = {g.nx, g.ny, g.nz};
  for (int c = 0; c < 3; ++c) {
    float* a = s->f[c];
    const int* e = g.e[c];
    for (int ax = 0; ax < 3; ++ax) {
      if (ax == c) continue;
      for (int side = 0; side < 2; ++side) {
        const int v = side ? n[ax] : 0;
        int lo[3] = {0, 0, 0}, hi[3] = {e[0], e[1], e[2]};
        lo[ax] = v;
        hi[ax] = v + 1;
        for (int k = lo[2]; k < hi[2]; ++k)
          for (int j = lo[1]; j < hi[1]; ++j)
            for (int i = lo[0]; i < hi[0]; ++i) a[AT(c, i, j, k)] = 0.0f;
      }
    }
  }
}

/* kernels.hpp:23-25 / :46-63, over the full H extents. */
void yo_faraday(yo_state* s, const yo_coeffs* c, int nthreads) {
  const geo g = make_geo(s);
  const float *ex = s->f[0], *ey = s->f[1], *ez = s->f[2];
  float *hx = s->f[3], *hy = s->f[4], *hz = s->f[5];
  /* hx: (nx+1) x ny x nz */
  OMP_FOR
  for (int k = 0; k < g.nz; ++k)
    for (int j = 0; j < g.ny; ++j) {
      const int64_t crow = CROW(j, k);
      for (int i = 0; i <= g.nx; ++i) {
        const int64_t cl = crow + (i < g.nx ? i : g.nx - 1);
        const float A = c->da ? c->da[cl] : c->da_s;
        const float C1 = c->db ? c->db[cl] : c->cdz[k];
        const float C2 = c->db ? c->db[cl] : c->cdy[j];
        const int64_t p = AT(3, i, j, k);
        const float d1 = ey[AT(1, i, j, k + 1)] - ey[AT(1, i, j, k)];
        const float d2 = ez[AT(2, i, j + 1, k)] - ez[AT(2, i, j, k)];
        const float t1 = C1 * d1;
        const float t2 = C2 * d2;
        const float inc = t1 - t2;
        hx[p] = A * hx[p] + inc;
      }
    }
  /* hy: nx x (ny+1) x nz */
  OMP_FOR
  for (int k = 0; k < g.nz; ++k)
    for (int j = 0; j <= g.ny; ++j) {
      const int64_t crow = CROW(j, k);
      for (int i = 0; i < g.nx; ++i) {
        const int64_t cl = crow + (i < g.nx ? i : g.nx - 1);
        const float A = c->da ? c->da[cl] : c->da_s;
        const float C1 = c->db ? c->db[cl] : c->cdx[i];
        const float C2 = c->db ? c->db[cl] : c->cdz[k];
        const int64_t p = AT(4, i, j, k);
        const float d1 = ez[AT(2, i + 1, j, k)] - ez[AT(2, i, j, k)];
        const float d2 = ex[AT(0, i, j, k + 1)] - ex[AT(0, i, j, k)];
        const float t1 = C1 * d1;
        const float t2 = C2 * d2;
        const float inc = t1 - t2;
        hy[p] = A * hy[p] + inc;
      }
    }
  /* hz: nx x ny x (nz+1) */
  OMP_FOR
  for (int k = 0; k <= g.nz; ++k)
    for (int j = 0; j < g.ny; ++j) {
      const int64_t crow = CROW(j, k);
      for (int i = 0; i < g.nx; ++i) {
        const int64_t cl = crow + (i < g.nx ? i : g.nx - 1);
        const float A = c->da ? c->da[cl] : c->da_s;
        const float C1 = c->db ? c->db[cl] : c->cdy[j];
        const float C2 = c->db ? c->db[cl] : c->cdx[i];
        const int64_t p = AT(5, i, j, k);
        const float d1 = ex[AT(0, i, j + 1, k)] - ex[AT(0, i, j, k)];
        const float d2 = ey[AT(1, i + 1, j, k)] - ey[AT(1, i, j, k)];
        const float t1 = C1 * d1;
        const float t2 = C2 * d2;
        const float inc = t1 - t2;
        hz[p] = A * hz[p] + inc;
      }
    }
}

/* plan_standard (schedule.hpp:171-210); inject_current (source.hpp:61-68). */
void yo_step(yo_state* s, const yo_coeffs* c, const yo_source* src, int nsrc,
             int64_t step, int nthreads) {
  const geo g = make_geo(s);
  yo_ampere(s, c, nthreads);
  yo_pec(s);
  for (int q = 0; q < nsrc; ++q) {
    if (step < 0 || step >= src[q].n) continue;
    const int cc = src[q].comp;
    s->f[cc][AT(cc, src[q].i, src[q].j, src[q].k)] += src[q].table[step];
  }
  yo_faraday(s, c, nthreads);
}

void yo_run(yo_state* s, const yo_coeffs* c, const yo_source* src, int nsrc,
            int64_t step0, int64_t nsteps, int nthreads) {
  for (int64_t t = 0; t < nsteps; ++t) yo_step(s, c, src, nsrc, step0 + t, nthreads);
}

uint64_t yo_digest(const yo_state* s) {
  uint64_t h = 1469598103934665603ull;
  for (int c = 0; c < 6; ++c) {
    const unsigned char* b = (const unsigned char*)s->f[c];
    const int64_t n = yo_comp_size(s->nx, s->ny, s->nz, c) * (int64_t)sizeof(float);
    for (int64_t i = 0; i < n; ++i) {
      h ^= b[i];
      h *= 1099511628211ull;
    }
  }
  return h;
}

void yo_fill_fields(yo_state* s, uint64_t seed, int nthreads) {
  for (int c = 0; c < 6; ++c) {
    const int64_t n = yo_comp_size(s->nx, s->ny, s->nz, c);
    float* a = s->f[c];
    OMP_FOR
    for (int64_t i = 0; i < n; ++i) a[i] = yb_field_value(seed, c, (uint64_t)i);
  }
}

void yo_make_cell_coeffs(int nx, int ny, int nz, int64_t eps_seed,
                         int64_t sigma_seed, float* ca, float* cb, float* da,
                         float* db, int nthreads) {
  const int64_t n = (int64_t)nx * ny * nz;
  const float S = yo_courant();
  OMP_FOR
  for (int64_t i = 0; i < n; ++i) {
    const yb_cell_coeffs q = yb_cell_coeffs_at(eps_seed, sigma_seed, (uint64_t)i, S);
    if (ca) ca[i] = q.ca;
    if (cb) cb[i] = q.cb;
    if (da) da[i] = q.da;
    if (db) db[i] = q.db;
  }
}

float yo_courant(void) {
  const uint32_t bits = YB_S_BITS;
  float f;
  memcpy(&f, &bits, sizeof f);
  return f;
}

void yo_gauss_table(float* out, int64_t n, double t0, double w) {
  for (int64_t i = 0; i < n; ++i) out[i] = yb_gauss_pulse(i, t0, w);
}
