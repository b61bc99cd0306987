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

// nz is the local slab depth; zoff/nzg place the slab in the global grid
// (single GPU: zoff = 0, nzg = nz). Arrays carry kGhost ghost planes below
// local plane 0 (base pointer = allocation + kGhost planes) and ghost planes
// nz (inside the node box) and nz+1 above; the two-step sweep needs both.
constexpr int kGhost = 2;
struct Geo {
  int nx, ny, nz;
  int PX, PY, PZ;
  long long plane;  // PX*PY
  long long total;  // floats per allocation: planes -2..nz+1 + 1 guard plane
  int zoff, nzg;    // global index of local plane 0, global cell count along z
};

__host__ __device__ __forceinline__ bool at_bottom(const Geo& g) { return g.zoff == 0; }
__host__ __device__ __forceinline__ bool at_top(const Geo& g) { return g.zoff + g.nz == g.nzg; }

struct SrcArgs {
  int n;
  int comp[kMaxSources], i[kMaxSources], j[kMaxSources], k[kMaxSources];
  float val[kMaxSources];   // increment at step n (the launch's first step)
  float val2[kMaxSources];  // increment at step n+1 (two-step sweeps)
  int act[kMaxSources];     // bit 0: active at step n, bit 1: active at step n+1
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

// Same with the leading coefficient A known to be exactly 1 when !HAS_A
// (uniform Ca / Da are only ever stored as the scalar 1, see
// yb_set_cell_coeffs): 1*v == v, so skipping the multiply is bit-identical.
template <bool HAS_A>
__device__ __forceinline__ float yee_upd_t(float A, float v, float C1, float a, float b, float C2, float c,
                                           float d) {
  if (HAS_A) return yee_upd(A, v, C1, a, b, C2, c, d);
  const float t1 = __fmul_rn(C1, __fsub_rn(a, b));
  const float t2 = __fmul_rn(C2, __fsub_rn(c, d));
  return __fadd_rn(v, __fsub_rn(t1, t2));
}

// Quiescent map (yb_set_quiescent_skip): bit (tile, plane) set once that
// tile-plane may hold a nonzero DoF in either state buffer. Tiles are the
// kTX x 8 sweep tiles (the last tile column / row also owns the i = nx /
// j = ny faces); planes are local, -kGhost .. nz + kGhost - 1.
struct QMap {
  unsigned* bits;  // nullptr: skipping off
  int words;       // 32-bit words per tile
  int ntx, nty;
};

__device__ __forceinline__ void qmap_mark(const QMap& q, int tile, int k) {
  const int b = k + kGhost;
  atomicOr(&q.bits[(size_t)tile * q.words + (b >> 5)], 1u << (b & 31));
}

// any bit set for tiles tx-1..tx+1 x ty-1..ty+1 and planes k0..k1?
__device__ __forceinline__ bool qmap_dirty(const QMap& q, int tx, int ty, int k0, int k1) {
  const int b0 = k0 + kGhost, b1 = k1 + kGhost;
  for (int y = max(ty - 1, 0); y <= min(ty + 1, q.nty - 1); ++y)
    for (int x = max(tx - 1, 0); x <= min(tx + 1, q.ntx - 1); ++x) {
      const unsigned* w = q.bits + (size_t)(y * q.ntx + x) * q.words;
      for (int wi = b0 >> 5; wi <= (b1 >> 5); ++wi) {
        unsigned m = __ldcg(w + wi);
        if (wi == (b0 >> 5)) m &= ~0u << (b0 & 31);
        if (wi == (b1 >> 5) && (b1 & 31) != 31) m &= (1u << ((b1 & 31) + 1)) - 1u;
        if (m) return true;
      }
    }
  return false;
}

// any source listed for this launch inside the box [x0,x1] x [y0,y1] x [k0,k1]
__device__ __forceinline__ bool src_in_box(const SrcArgs& s, int x0, int x1, int y0, int y1, int k0, int k1) {
  for (int q = 0; q < s.n; ++q)
    if (s.act[q] && s.i[q] >= x0 && s.i[q] <= x1 && s.j[q] >= y0 && s.j[q] <= y1 && s.k[q] >= k0 &&
        s.k[q] <= k1)
      return true;
  return false;
}

__device__ __forceinline__ bool nonzero4(float4 v) {
  return (__float_as_uint(v.x) | __float_as_uint(v.y) | __float_as_uint(v.z) | __float_as_uint(v.w)) != 0u;
}

constexpr int kSkipItem = 1 << 30;  // item_q flag: the item is quiescent, no data staged

__device__ __forceinline__ long long gidx(const Geo& g, int i, int j, int k) {
  return ((long long)k * g.PY + j) * g.PX + i;
}

__device__ __forceinline__ float coefA(const float* cell, float s, long long p) {
  return cell ? cell[p] : s;
}
__device__ __forceinline__ float coefB(const float* cell, const float* axis, int ax, long long p) {
  return cell ? cell[p] : axis[ax];
}

// DoFs on the three upper faces (i=nx, j=ny, k=nz) that the cell-box sweep
// does not own. Tangential E there is PEC (written +0); the normal H (hx at
// i=nx, hy at j=ny, hz at k=nz) reads only those PEC zeros, so its update is
// Da*h + (Db*(0-0) - Db*(0-0)), computed in exactly that form. Reads `in`,
// writes `out` (disjoint from the sweep's writes). Per-cell Da / Db are read
// at the clamped cell (i, j, k limited to the cell box) — the value the
// arrays' clamped duplicates at i=nx / j=ny / k=nz hold — so the face update
// does not depend on those duplicates being filled yet (yb_run_streamed fills
// them after the run).
// Owned node planes of the slab: 0..nz-1, plus plane nz at the global top.
__device__ __forceinline__ int face_nk(const Geo& g) { return at_top(g) ? g.nz + 1 : g.nz; }

__device__ __forceinline__ long long face_points(const Geo& g) {
  const int nk = face_nk(g);
  return (long long)(g.ny + 1) * nk + (long long)(g.nx + 1) * nk +
         (at_top(g) ? (long long)(g.nx + 1) * (g.ny + 1) : 0LL);
}

__device__ __forceinline__ void face_point(const Geo& g, const float* const* in,
                                           float* const* out, const CoefArgs& co, long long t) {
  const int nk = face_nk(g);
  const long long nxf = (long long)(g.ny + 1) * nk;
  const long long nyf = (long long)(g.nx + 1) * nk;
  if (t < nxf) {
    const int j = (int)(t % (g.ny + 1)), k = (int)(t / (g.ny + 1)), i = g.nx;
    const long long p = gidx(g, i, j, k), pc = p - 1;
    if (j < g.ny) out[1][p] = 0.0f;
    if (k < g.nz) out[2][p] = 0.0f;
    if (j < g.ny && k < g.nz)
      out[3][p] = yee_upd(coefA(co.cell[2], co.da_s, pc), in[3][p], coefB(co.cell[3], co.cdz_h, k, pc),
                          0.0f, 0.0f, coefB(co.cell[3], co.cdy_h, j, pc), 0.0f, 0.0f);
  } else if (t < nxf + nyf) {
    const long long u = t - nxf;
    const int i = (int)(u % (g.nx + 1)), k = (int)(u / (g.nx + 1)), j = g.ny;
    const long long p = gidx(g, i, j, k), pc = p - g.PX;
    if (i < g.nx) out[0][p] = 0.0f;
    if (k < g.nz) out[2][p] = 0.0f;
    if (i < g.nx && k < g.nz)
      out[4][p] = yee_upd(coefA(co.cell[2], co.da_s, pc), in[4][p], coefB(co.cell[3], co.cdx_h, i, pc),
                          0.0f, 0.0f, coefB(co.cell[3], co.cdz_h, k, pc), 0.0f, 0.0f);
  } else {
    const long long u = t - nxf - nyf;
    const int i = (int)(u % (g.nx + 1)), j = (int)(u / (g.nx + 1)), k = g.nz;
    const long long p = gidx(g, i, j, k), pc = p - (long long)g.PX * g.PY;
    if (i < g.nx) out[0][p] = 0.0f;
    if (j < g.ny) out[1][p] = 0.0f;
    if (i < g.nx && j < g.ny)
      out[5][p] = yee_upd(coefA(co.cell[2], co.da_s, pc), in[5][p], coefB(co.cell[3], co.cdy_h, j, pc),
                          0.0f, 0.0f, coefB(co.cell[3], co.cdx_h, i, pc), 0.0f, 0.0f);
  }
}

}  // namespace yb
