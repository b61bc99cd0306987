// yb_device.cuh — device-side layout, argument structs and shared helpers.
//
// Device layout: every component and every
// per-cell coefficient array lives on ONE padded node box
//     x: PX = round_up(nx+1, 32) floats (128-byte rows),  y: PY = ny+1,  z: PZ = nz+1
// at index (k*PY + j)*PX + i, so the same (i,j,k) addresses the same Yee
// cell in all arrays. Positions outside a component's extents
// (staggering.hpp:34-39) are never written and stay +0.0. Per-cell
// coefficients hold clamped duplicates at i=nx, j=ny, k=nz (the DoF's own
// cell, clamped to the grid: include/yeeb200_inputs.h).
#pragma once

#include <cstdint>

namespace yb {

constexpr int kMaxSources = 8;

struct Geo {
  int nx, ny, nz;
  int PX, PY, PZ;
  long long plane;  // PX*PY
  long long total;  // floats per array incl. guard
};

struct SrcArgs {
  int n;
  int comp[kMaxSources], i[kMaxSources], j[kMaxSources], k[kMaxSources];
  float val[kMaxSources];
};

// Coefficients as seen by a kernel: per-cell arrays (nullptr if not cell
// mode), scalars for Ca/Da, per-axis arrays for Cb/Db (E set and H set).
struct CoefArgs {
  const float* cell[4];  // Ca, Cb, Da, Db (padded node box) or nullptr
  float ca_s, da_s;
  const float *cdx_e, *cdy_e, *cdz_e;
  const float *cdx_h, *cdy_h, *cdz_h;
};

struct Fields {
  float* f[6];
};

// v' = A*v + (C1*(a-b) - C2*(c-d)): reference operand order
// (kernels.hpp:10-25), every operation individually rounded (never
// contracted into FMA) so the result is bit-identical to the CPU oracle.
__device__ __forceinline__ float yee_upd(float A, float v, float C1, float a, float b, float C2,
                                         float c, float d) {
  const float t1 = __fmul_rn(C1, __fsub_rn(a, b));
  const float t2 = __fmul_rn(C2, __fsub_rn(c, d));
  return __fadd_rn(__fmul_rn(A, v), __fsub_rn(t1, t2));
}

__device__ __forceinline__ long long gidx(const Geo& g, int i, int j, int k) {
  return ((long long)k * g.PY + j) * g.PX + i;
}

}  // namespace yb
