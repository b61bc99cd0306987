/*
 * yee_oracle.h — CPU ORACLE (test infrastructure only).
 *
 * A plain-C restatement of the reference yeeblock Standard step
 * (/root/reference/proj/include/yeeblock), extended with per-cell
 * Ca/Cb/Da/Db coefficients. It is the checker for the CUDA path: only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * legs may load it. The product library (libyeeb200.so) never links or
 * calls it.
 *
 * Parity pinning: with Ca = Da = 1 and Cb/Db taken from the reference's 1D
 * cdx/cdy/cdz arrays it is bit-identical to the unmodified reference kernels
 * (checked against oracle/_ref, the reference headers compiled by
 * oracle/Makefile, and against tests/golden/ fixtures generated from it).
 *
 * Storage is the reference's dense Array3 layout per component: extents
 * from staggering.hpp:34-39, index (k*ny + j)*nx + i (array3.hpp:104-107).
 */
#ifndef YEE_ORACLE_H
#define YEE_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { YO_EX = 0, YO_EY, YO_EZ, YO_HX, YO_HY, YO_HZ };

typedef struct {
  int nx, ny, nz;  /* cells */
  float *f[6];     /* ex..hz, dense per-component arrays */
} yo_state;

/*
 * Coefficient set. Ca/Da: per-cell array (nx*ny*nz, dense cell order) or,
 * when NULL, the scalar ca_s/da_s. Cb/Db: per-cell array or, when NULL, the
 * reference's per-axis arrays cdx[nx], cdy[ny], cdz[nz] (grid.hpp:79-103).
 * Per-cell values of DoF (i,j,k) are read at the cell (clamp(i,0,nx-1),
 * clamp(j,0,ny-1), clamp(k,0,nz-1)).
 */
typedef struct {
  const float *ca, *cb, *da, *db;
  float ca_s, da_s;
  const float *cdx, *cdy, *cdz;
} yo_coeffs;

/* Point soft source: comp(i,j,k) += table[step] for step < n. */
typedef struct {
  int comp, i, j, k;
  const float* table;
  int64_t n;
} yo_source;

void yo_comp_extents(int nx, int ny, int nz, int comp, int ext[3]);
int64_t yo_comp_size(int nx, int ny, int nz, int comp);

/* Ampere over curl_updatable_box (kernels.hpp:129-135, :27-44). */
void yo_ampere(yo_state* s, const yo_coeffs* c, int nthreads);
/* Tangential-E zeroing on the six faces (kernels.hpp:147-155). */
void yo_pec(yo_state* s);
/* Faraday over the full H extents (kernels.hpp:138-144, :46-63). */
void yo_faraday(yo_state* s, const yo_coeffs* c, int nthreads);
/* One Standard step (schedule.hpp:171-210): Ampere, PEC, sources, Faraday.
 * `step` = completed steps before this one (runner.hpp:103-104). */
void yo_step(yo_state* s, const yo_coeffs* c, const yo_source* src, int nsrc,
             int64_t step, int nthreads);
void yo_run(yo_state* s, const yo_coeffs* c, const yo_source* src, int nsrc,
            int64_t step0, int64_t nsteps, int nthreads);

/* FNV-1a-64 over raw bytes Ex..Hz (fields.hpp:151-166). */
uint64_t yo_digest(const yo_state* s);

/* Seeded inputs (include/yeeb200_inputs.h). */
void yo_fill_fields(yo_state* s, uint64_t seed, int nthreads);
void yo_make_cell_coeffs(int nx, int ny, int nz, int64_t eps_seed,
                         int64_t sigma_seed, float* ca, float* cb, float* da,
                         float* db, int nthreads);
float yo_courant(void);
void yo_gauss_table(float* out, int64_t n, double t0, double w);

#ifdef __cplusplus
}
#endif

#endif
