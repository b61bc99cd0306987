// yb_basic.cu — per-DoF kernels (the NAIVE variant and the reference range
// operations), the boundary-face kernel of the FUSED variant, and the
// device-side seeded initialisers.
//
// Reference semantics followed (paths under /root/reference/proj/include/yeeblock):
//   Ampere  update_e_dof kernels.hpp:27-44 over curl_updatable_box staggering.hpp:70-77
//   Faraday update_h_dof kernels.hpp:46-63 over comp_extents staggering.hpp:44-49
//   PEC     apply_pec_boundary kernels.hpp:146-155 / pec_boxes staggering.hpp:81-86
//   Source  inject_current source.hpp:61-68
#include <cuda_runtime.h>

#include <algorithm>

#include "../../include/yeeb200_inputs.h"
#include "yb_device.cuh"
#include "yb_launch.h"
#include "yb_ptx.cuh"

namespace yb {

namespace {

struct Box {
  int xlo, xhi, ylo, yhi, zlo, zhi;
};

__device__ __forceinline__ bool in_box(const Box& b, int i, int j, int k) {
  return i >= b.xlo && i < b.xhi && j >= b.ylo && j < b.yhi && k >= b.zlo && k < b.zhi;
}

// One thread per node-box point (i,j,k), all three E components.
__global__ void k_naive_ampere(Geo g, Fields F, CoefArgs co, Box b) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y;
  const int k = blockIdx.z;
  if (i > g.nx || !in_box(b, i, j, k)) return;
  const long long p = gidx(g, i, j, k);
  float *ex = F.f[0], *ey = F.f[1], *ez = F.f[2];
  const float *hx = F.f[3], *hy = F.f[4], *hz = F.f[5];
  const float A = coefA(co.cell[0], co.ca_s, p);
  const bool ji = j >= 1 && j < g.ny, ki = k >= 1 && k < g.nz, ii = i >= 1 && i < g.nx;
  if (i < g.nx && ji && ki)  // ex: (h,n,n)
    ex[p] = yee_upd(A, ex[p], coefB(co.cell[1], co.cdy_e, j, p), hz[p], hz[p - g.PX],
                    coefB(co.cell[1], co.cdz_e, k, p), hy[p], hy[p - g.plane]);
  if (ii && j < g.ny && ki)  // ey: (n,h,n)
    ey[p] = yee_upd(A, ey[p], coefB(co.cell[1], co.cdz_e, k, p), hx[p], hx[p - g.plane],
                    coefB(co.cell[1], co.cdx_e, i, p), hz[p], hz[p - 1]);
  if (ii && ji && k < g.nz)  // ez: (n,n,h)
    ez[p] = yee_upd(A, ez[p], coefB(co.cell[1], co.cdx_e, i, p), hy[p], hy[p - 1],
                    coefB(co.cell[1], co.cdy_e, j, p), hx[p], hx[p - g.PX]);
}

__global__ void k_naive_faraday(Geo g, Fields F, CoefArgs co, Box b) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y;
  const int k = blockIdx.z;
  if (i > g.nx || !in_box(b, i, j, k)) return;
  const long long p = gidx(g, i, j, k);
  const float *ex = F.f[0], *ey = F.f[1], *ez = F.f[2];
  float *hx = F.f[3], *hy = F.f[4], *hz = F.f[5];
  const float A = coefA(co.cell[2], co.da_s, p);
  if (j < g.ny && k < g.nz)  // hx: (nx+1) x ny x nz
    hx[p] = yee_upd(A, hx[p], coefB(co.cell[3], co.cdz_h, k, p), ey[p + g.plane], ey[p],
                    coefB(co.cell[3], co.cdy_h, j, p), ez[p + g.PX], ez[p]);
  if (i < g.nx && k < g.nz)  // hy: nx x (ny+1) x nz
    hy[p] = yee_upd(A, hy[p], coefB(co.cell[3], co.cdx_h, i, p), ez[p + 1], ez[p],
                    coefB(co.cell[3], co.cdz_h, k, p), ex[p + g.plane], ex[p]);
  if (i < g.nx && j < g.ny)  // hz: nx x ny x (nz+1)
    hz[p] = yee_upd(A, hz[p], coefB(co.cell[3], co.cdy_h, j, p), ex[p + g.PX], ex[p],
                    coefB(co.cell[3], co.cdx_h, i, p), ey[p + 1], ey[p]);
}

// Tangential E on the six faces := +0 (node-axis planes 0 and n).
__global__ void k_naive_pec(Geo g, Fields F) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y;
  const int k = blockIdx.z;
  if (i > g.nx) return;
  const long long p = gidx(g, i, j, k);
  const bool bi = i == 0 || i == g.nx, bj = j == 0 || j == g.ny, bk = k == 0 || k == g.nz;
  if (i < g.nx && (bj || bk)) F.f[0][p] = 0.0f;
  if (j < g.ny && (bi || bk)) F.f[1][p] = 0.0f;
  if (k < g.nz && (bi || bj)) F.f[2][p] = 0.0f;
}

__global__ void k_sources(Geo g, Fields F, SrcArgs s) {
  if (threadIdx.x != 0) return;
  for (int q = 0; q < s.n; ++q) {
    float* a = F.f[s.comp[q]];
    const long long p = gidx(g, s.i[q], s.j[q], s.k[q]);
    a[p] = __fadd_rn(a[p], s.val[q]);
  }
}

// FUSED-variant companion: the DoFs on the three upper faces (i=nx, j=ny,
// k=nz) that the cell-box sweep does not own. Tangential E there is PEC
// (written +0); the normal H (hx at i=nx, hy at j=ny, hz at k=nz) reads only
// those PEC zeros, so its update is Da*h + (Db*(0-0) - Db*(0-0)), computed
// in exactly that form. Reads `in`, writes `out` (disjoint from the sweep).
__global__ void k_faces(Geo g, Fields in, Fields out, CoefArgs co) {
  const long long total = face_points(g);
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x)
    face_point(g, in.f, out.f, co, t);
}

// Extents of component c on the GLOBAL grid (nz -> nzg).
__device__ __forceinline__ void comp_ext(const Geo& g, int c, int e[3]) {
  const int n[3] = {g.nx, g.ny, g.nzg};
  const int axis = c % 3;
  for (int a = 0; a < 3; ++a) {
    const bool node = c < 3 ? (a != axis) : (a == axis);
    e[a] = n[a] + (node ? 1 : 0);
  }
}

// Seeded fields over each component's extents, hashed by the GLOBAL dense
// reference index, so any z-slab partition generates the same state.
__global__ void k_fill_fields(Geo g, Fields F, uint64_t seed) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y;
  const int k = blockIdx.z;
  if (i > g.nx) return;
  const long long p = gidx(g, i, j, k);
  const int kg = k + g.zoff;
#pragma unroll
  for (int c = 0; c < 6; ++c) {
    int e[3];
    comp_ext(g, c, e);
    if (i < e[0] && j < e[1] && kg < e[2]) {
      const uint64_t dense = ((uint64_t)kg * e[1] + j) * e[0] + i;
      F.f[c][p] = yb_field_value(seed, c, dense);
    }
  }
}

// Pinned medium over the node box and the ghost planes (local planes
// -kGhost..nz+1) with the clamped GLOBAL cell index.
__global__ void k_medium(Geo g, float* ca, float* cb, float* da, float* db, long long eps_seed,
                         long long sigma_seed, float S) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y;
  const int k = (int)blockIdx.z - kGhost;
  if (i > g.nx) return;
  const int ci = min(i, g.nx - 1), cj = min(j, g.ny - 1), ck = max(0, min(k + g.zoff, g.nzg - 1));
  const uint64_t cell = ((uint64_t)ck * g.ny + cj) * g.nx + ci;
  const yb_cell_coeffs q = yb_cell_coeffs_at(eps_seed, sigma_seed, cell, S);
  const long long p = gidx(g, i, j, k);
  if (ca) ca[p] = q.ca;
  if (cb) cb[p] = q.cb;
  if (da) da[p] = q.da;
  if (db) db[p] = q.db;
}

// After a dense upload of cell planes kmin..kmax into [0,nx)x[0,ny): fill the
// clamped duplicates at i=nx, j=ny and on the other planes of -kGhost..nz+1.
__global__ void k_clamp_fill(Geo g, float* a, int kmin, int kmax) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y;
  const int k = (int)blockIdx.z - kGhost;
  if (i > g.nx) return;
  if (i < g.nx && j < g.ny && k >= kmin && k <= kmax) return;
  a[gidx(g, i, j, k)] = a[gidx(g, min(i, g.nx - 1), min(j, g.ny - 1), max(kmin, min(k, kmax)))];
}

// Dense (reference Array3 layout, extents e0 x e1 x e2) <-> padded node box.
__global__ void k_scatter_dense(Geo g, int e0, int e1, int e2, const float* __restrict__ dense,
                                float* __restrict__ padded) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y;
  const int k = blockIdx.z;
  if (i >= e0 || j >= e1 || k >= e2) return;
  padded[gidx(g, i, j, k)] = dense[((long long)k * e1 + j) * e0 + i];
}

__global__ void k_gather_dense(Geo g, int e0, int e1, int e2, const float* __restrict__ padded,
                               float* __restrict__ dense) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y;
  const int k = blockIdx.z;
  if (i >= e0 || j >= e1 || k >= e2) return;
  dense[((long long)k * e1 + j) * e0 + i] = padded[gidx(g, i, j, k)];
}

// *flag := 0 if any element's bit pattern differs from a[0].
__global__ void k_all_equal(const float* __restrict__ a, long long n, int* flag) {
  const unsigned v0 = __float_as_uint(a[0]);
  bool same = true;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n;
       t += (long long)gridDim.x * blockDim.x)
    same &= __float_as_uint(a[t]) == v0;
  if (!__all_sync(0xffffffffu, same) && (threadIdx.x & 31) == 0) atomicExch(flag, 0);
}

// One block per (tile, plane): 8 warps over the tile's rows, lanes over its
// columns (float4); the last tile column / row also covers the padding and
// the i = nx / j = ny faces.
__global__ void __launch_bounds__(256) k_qscan(Geo g, Fields A, Fields Bf, QMap q, int k0) {
  const int tile = blockIdx.x, k = k0 + (int)blockIdx.y;
  const int tx = tile % q.ntx, ty = tile / q.ntx;
  const int x0 = tx * kTX, y0 = ty * 8;
  const int xe = tx == q.ntx - 1 ? g.PX : x0 + kTX, ye = ty == q.nty - 1 ? g.PY : y0 + 8;
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  bool nz = false;
  for (int j = y0 + w; j < ye; j += 8)
    for (int i = x0 + 4 * l; i < xe; i += 128) {
      const long long p = ((long long)k * g.PY + j) * g.PX + i;
#pragma unroll
      for (int c = 0; c < 6; ++c)
        nz |= nonzero4(*reinterpret_cast<const float4*>(A.f[c] + p)) |
              nonzero4(*reinterpret_cast<const float4*>(Bf.f[c] + p));
    }
  if (__syncthreads_or(nz) && threadIdx.x == 0) qmap_mark(q, tile, k);
}

// Peer halo push: blockIdx.y = direction (0 down, 1 up); float4 copies over
// nplanes x 6 components x one padded plane each.
__global__ void k_peer_copy(Geo g, PeerCopy d0, PeerCopy d1) {
  const PeerCopy& d = blockIdx.y == 0 ? d0 : d1;
  const long long per = g.plane / 4;  // float4 per plane (PX is a multiple of 32)
  const long long n = per * 6 * d.nplanes;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x) {
    const long long q = t / per, e = t - q * per;
    const int c = (int)(q % 6), k = (int)(q / 6);
    const float4 v = reinterpret_cast<const float4*>(d.src[c] + (long long)(d.src_k0 + k) * g.plane)[e];
    reinterpret_cast<float4*>(d.dst[c] + (long long)(d.dst_k0 + k) * g.plane)[e] = v;
  }
}

__global__ void k_peer_signal(unsigned* f0, unsigned* f1, unsigned epoch) {
  __threadfence_system();
  if (f0) asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(f0), "r"(epoch) : "memory");
  if (f1) asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(f1), "r"(epoch) : "memory");
}

__global__ void k_peer_wait(const unsigned* flags, unsigned need0, unsigned need1, int* err,
                            unsigned long long wait_ns) {
  const unsigned long long t0 = globaltimer_ns();
  for (;;) {
    unsigned a, b;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(a) : "l"(flags) : "memory");
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(b) : "l"(flags + 1) : "memory");
    if (a >= need0 && b >= need1) return;
    if (globaltimer_ns() - t0 > wait_ns) {  // the neighbour never signalled: report, do not hang
      const bool lo = a < need0;
      wait_timed_out(err, WAIT_PEER, -1, lo ? 0 : 1, lo ? a : b, lo ? need0 : need1);
      return;
    }
    __nanosleep(256);
  }
}

// Halo planes <-> exchange buffer, one launch for all planes (blockIdx.y = plane).
__global__ void k_halo_copy(Geo g, HaloList l, float* ext, bool pack) {
  const long long per = g.plane / 4;  // float4 per plane (PX is a multiple of 32)
  float4* e = reinterpret_cast<float4*>(ext + (long long)blockIdx.y * g.plane);
  float4* d = reinterpret_cast<float4*>(l.plane[blockIdx.y]);
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < per; t += (long long)gridDim.x * blockDim.x) {
    if (pack)
      e[t] = d[t];
    else
      d[t] = e[t];
  }
}

__global__ void k_fill_value(float* p, long long n, float v) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x)
    p[t] = v;
}

// Point probes: out[q] = field[comp[q]][off[q]] (sample_probes, probe.hpp:36-51).
__global__ void k_probes(Fields F, ProbeArgs pa, float* out) {
  const int q = threadIdx.x;
  if (q < pa.n) out[q] = F.f[pa.comp[q]][pa.off[q]];
}

// Leapfrog invariant (total_energy, fields.hpp:116-146): per-(component,
// block) partial sums in double with a fixed tree, then one fixed-order sum.
// dof volume = ((1 * w_x) * w_y) * w_z as in dof_volume (fields.hpp:96-105);
// a term is (V * e) * e for E and (V * prev) * now for H.
__global__ void __launch_bounds__(256) k_energy(Geo g, Fields F, const float* p0, const float* p1,
                                                const float* p2, const double* w, double* partial) {
  const int c = blockIdx.y;
  const bool top = at_top(g);
  const int planes = (c == 0 || c == 1 || c == 5) ? g.nz + (top ? 1 : 0) : g.nz;  // owned planes
  const double* wn[3] = {w, w + 2 * g.nx + 1, w + 2 * g.nx + 2 * g.ny + 2};
  const double* wc[3] = {w + g.nx + 1, w + 2 * g.nx + g.ny + 2, w + 2 * g.nx + 2 * g.ny + 2 + g.nz + 1};
  const bool node[3] = {c < 3 ? c != 0 : c == 3, c < 3 ? c != 1 : c == 4, c < 3 ? c != 2 : c == 5};
  const int e[3] = {g.nx + node[0], g.ny + node[1], g.nz + node[2]};
  const double* wx = node[0] ? wn[0] : wc[0];
  const double* wy = node[1] ? wn[1] : wc[1];
  const double* wz = node[2] ? wn[2] : wc[2];
  const float* a = F.f[c];
  const float* pv = c == 3 ? p0 : (c == 4 ? p1 : p2);
  double acc = 0.0;
  const long long rows = (long long)planes * e[1];
  for (long long r = blockIdx.x; r < rows; r += gridDim.x) {
    const int k = (int)(r / e[1]), j = (int)(r % e[1]);
    const double vyz_y = wy[j], vz = wz[k];
    const long long base = ((long long)k * g.PY + j) * g.PX;
    for (int i = threadIdx.x; i < e[0]; i += blockDim.x) {
      const double v = __dmul_rn(__dmul_rn(__dmul_rn(1.0, wx[i]), vyz_y), vz);
      const double now = (double)a[base + i];
      const double t = c < 3 ? __dmul_rn(__dmul_rn(v, now), now) : __dmul_rn(__dmul_rn(v, (double)pv[base + i]), now);
      acc = __dadd_rn(acc, t);
    }
  }
  __shared__ double red[256];
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int h = 128; h > 0; h >>= 1) {
    if (threadIdx.x < h) red[threadIdx.x] = __dadd_rn(red[threadIdx.x], red[threadIdx.x + h]);
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[c * gridDim.x + blockIdx.x] = red[0];
}

__global__ void k_energy_final(const double* partial, int n, double* out) {
  double s = 0.0;
  for (int q = 0; q < n; ++q) s = __dadd_rn(s, partial[q]);
  *out = s;
}

dim3 node_grid(const Geo& g, int bx) { return dim3((g.nx + 1 + bx - 1) / bx, g.ny + 1, g.nz + 1); }
// node box plus the ghost planes: local planes -kGhost..nz+1
dim3 ghost_grid(const Geo& g, int bx) {
  return dim3((g.nx + 1 + bx - 1) / bx, g.ny + 1, g.nz + 2 + kGhost);
}

}  // namespace

cudaError_t launch_naive_ampere(const Geo& g, const Fields& F, const CoefArgs& co, const int* box,
                                cudaStream_t st) {
  const Box b{box[0], box[1], box[2], box[3], box[4], box[5]};
  k_naive_ampere<<<node_grid(g, 128), 128, 0, st>>>(g, F, co, b);
  return cudaGetLastError();
}

cudaError_t launch_naive_faraday(const Geo& g, const Fields& F, const CoefArgs& co, const int* box,
                                 cudaStream_t st) {
  const Box b{box[0], box[1], box[2], box[3], box[4], box[5]};
  k_naive_faraday<<<node_grid(g, 128), 128, 0, st>>>(g, F, co, b);
  return cudaGetLastError();
}

cudaError_t launch_naive_pec(const Geo& g, const Fields& F, cudaStream_t st) {
  k_naive_pec<<<node_grid(g, 128), 128, 0, st>>>(g, F);
  return cudaGetLastError();
}

cudaError_t launch_sources(const Geo& g, const Fields& F, const SrcArgs& s, cudaStream_t st) {
  k_sources<<<1, 32, 0, st>>>(g, F, s);
  return cudaGetLastError();
}

cudaError_t launch_faces(const Geo& g, const Fields& in, const Fields& out, const CoefArgs& co,
                         int num_sms, cudaStream_t st) {
  const long long total = (long long)(g.ny + 1) * (g.nz + 1) + (long long)(g.nx + 1) * (g.nz + 1) +
                          (long long)(g.nx + 1) * (g.ny + 1);
  long long blocks = (total + 255) / 256;
  if (blocks > 4LL * num_sms) blocks = 4LL * num_sms;
  k_faces<<<(unsigned)blocks, 256, 0, st>>>(g, in, out, co);
  return cudaGetLastError();
}

cudaError_t launch_fill_fields(const Geo& g, const Fields& F, uint64_t seed, cudaStream_t st) {
  k_fill_fields<<<node_grid(g, 128), 128, 0, st>>>(g, F, seed);
  return cudaGetLastError();
}

cudaError_t launch_medium(const Geo& g, float* ca, float* cb, float* da, float* db,
                          long long eps_seed, long long sigma_seed, float S, cudaStream_t st) {
  k_medium<<<ghost_grid(g, 128), 128, 0, st>>>(g, ca, cb, da, db, eps_seed, sigma_seed, S);
  return cudaGetLastError();
}

cudaError_t launch_scatter_dense(const Geo& g, const int* e, const float* dense, float* padded,
                                 cudaStream_t st) {
  k_scatter_dense<<<dim3((e[0] + 127) / 128, e[1], e[2]), 128, 0, st>>>(g, e[0], e[1], e[2], dense,
                                                                        padded);
  return cudaGetLastError();
}

cudaError_t launch_gather_dense(const Geo& g, const int* e, const float* padded, float* dense,
                                cudaStream_t st) {
  k_gather_dense<<<dim3((e[0] + 127) / 128, e[1], e[2]), 128, 0, st>>>(g, e[0], e[1], e[2], padded,
                                                                       dense);
  return cudaGetLastError();
}

cudaError_t launch_qscan(const Geo& g, const Fields& a, const Fields& b, const QMap& q, int k0, int k1,
                         cudaStream_t st) {
  if (k1 < k0) return cudaSuccess;
  k_qscan<<<dim3(q.ntx * q.nty, k1 - k0 + 1), 256, 0, st>>>(g, a, b, q, k0);
  return cudaGetLastError();
}

cudaError_t launch_peer_copy(const Geo& g, const PeerCopy& down, const PeerCopy& up, cudaStream_t st) {
  if (!down.nplanes && !up.nplanes) return cudaSuccess;
  k_peer_copy<<<dim3(296, 2), 256, 0, st>>>(g, down, up);
  return cudaGetLastError();
}

cudaError_t launch_peer_signal(unsigned* flag_down, unsigned* flag_up, unsigned epoch, cudaStream_t st) {
  k_peer_signal<<<1, 1, 0, st>>>(flag_down, flag_up, epoch);
  return cudaGetLastError();
}

cudaError_t launch_peer_wait(const unsigned* flags, unsigned need0, unsigned need1, int* err,
                             unsigned long long wait_ns, cudaStream_t st) {
  k_peer_wait<<<1, 1, 0, st>>>(flags, need0, need1, err, wait_ns);
  return cudaGetLastError();
}

cudaError_t launch_halo_copy(const Geo& g, const HaloList& l, float* ext, bool pack, cudaStream_t st) {
  if (l.n == 0) return cudaSuccess;
  const long long per = g.plane / 4;
  const int bx = (int)std::min<long long>((per + 255) / 256, 148);
  k_halo_copy<<<dim3(bx, l.n), 256, 0, st>>>(g, l, ext, pack);
  return cudaGetLastError();
}

cudaError_t launch_fill_value(float* p, long long n, float v, cudaStream_t st) {
  k_fill_value<<<592, 256, 0, st>>>(p, n, v);
  return cudaGetLastError();
}

cudaError_t launch_probes(const Fields& F, const ProbeArgs& pa, float* out, cudaStream_t st) {
  k_probes<<<1, 64, 0, st>>>(F, pa, out);
  return cudaGetLastError();
}

cudaError_t launch_energy(const Geo& g, const Fields& F, const float* const* prev_h, const double* w,
                          double* partial, double* out, cudaStream_t st) {
  k_energy<<<dim3(kEnergyBlocks, 6), 256, 0, st>>>(g, F, prev_h[0], prev_h[1], prev_h[2], w, partial);
  k_energy_final<<<1, 1, 0, st>>>(partial, 6 * kEnergyBlocks, out);
  return cudaGetLastError();
}

cudaError_t launch_all_equal(const float* a, long long n, int* flag, int num_sms, cudaStream_t st) {
  k_all_equal<<<num_sms * 4, 256, 0, st>>>(a, n, flag);
  return cudaGetLastError();
}

cudaError_t launch_clamp_fill(const Geo& g, float* a, int kmin, int kmax, cudaStream_t st) {
  k_clamp_fill<<<ghost_grid(g, 128), 128, 0, st>>>(g, a, kmin, kmax);
  return cudaGetLastError();
}

}  // namespace yb
