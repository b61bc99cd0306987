// yb_hostops.cu — the reference's free per-box operations on a caller's
// FieldSet<Real> in HOST memory, for Real = float or double (the reference
// is templated on Real and its own unit tests run in double):
//   update_e_box / update_h_box / zero_box   kernels.hpp:78-111
//   apply_ampere_range / apply_faraday_range kernels.hpp:129-144
//   apply_pec_boundary                       kernels.hpp:147-155 (pec_boxes, staggering.hpp:81-86)
//   total_energy                             fields.hpp:116-146
// The arrays stay in the reference's dense Array3 layout (array3.hpp:104-107)
// on the device too: these are per-DoF kernels, one thread per DoF of the
// box, with the update expressions of kernels.hpp:27-63 in the reference's
// operand order (difference, scale, signed combination, accumulation) as
// explicit round-to-nearest intrinsics — bit-identical to the reference in
// either precision. The device-resident fp32 hot path is yb_tb2.cu /
// yb_fused.cu; these exist so that reference code holding its state in
// host FieldSets runs unchanged.
#include <cuda_runtime.h>

#include "yb_launch.h"

namespace yb {
namespace {

template <class T>
struct Rn;
template <>
struct Rn<float> {
  static __device__ __forceinline__ float sub(float a, float b) { return __fsub_rn(a, b); }
  static __device__ __forceinline__ float mul(float a, float b) { return __fmul_rn(a, b); }
  static __device__ __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
};
template <>
struct Rn<double> {
  static __device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
  static __device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
  static __device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
};

// v += C1*(a-b) - C2*(c-d)
template <class T>
__device__ __forceinline__ T upd(T v, T C1, T a, T b, T C2, T c, T d) {
  using R = Rn<T>;
  return R::add(v, R::sub(R::mul(C1, R::sub(a, b)), R::mul(C2, R::sub(c, d))));
}

__device__ __forceinline__ long long at(const HostExt& x, int c, int i, int j, int k) {
  return ((long long)k * x.e[c][1] + j) * x.e[c][0] + i;
}

// One component over a box: op 0 = E update, 1 = H update, 2 = zero.
template <class T>
__global__ void k_box(HostFields<T> f, HostExt x, int op, int comp, HostBox b) {
  const int nxb = b.xhi - b.xlo, nyb = b.yhi - b.ylo;
  const long long n = (long long)nxb * nyb * (b.zhi - b.zlo);
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x) {
    const int i = b.xlo + (int)(t % nxb);
    const int j = b.ylo + (int)((t / nxb) % nyb);
    const int k = b.zlo + (int)(t / ((long long)nxb * nyb));
    T* const* F = f.f;
    const T *cdx = f.cd[0], *cdy = f.cd[1], *cdz = f.cd[2];
    if (op == 2) {
      F[comp][at(x, comp, i, j, k)] = T(0);
      continue;
    }
    switch (comp) {  // kernels.hpp:27-63
      case 0: {
        T& v = F[0][at(x, 0, i, j, k)];
        v = upd(v, cdy[j], F[5][at(x, 5, i, j, k)], F[5][at(x, 5, i, j - 1, k)], cdz[k], F[4][at(x, 4, i, j, k)],
                F[4][at(x, 4, i, j, k - 1)]);
        break;
      }
      case 1: {
        T& v = F[1][at(x, 1, i, j, k)];
        v = upd(v, cdz[k], F[3][at(x, 3, i, j, k)], F[3][at(x, 3, i, j, k - 1)], cdx[i], F[5][at(x, 5, i, j, k)],
                F[5][at(x, 5, i - 1, j, k)]);
        break;
      }
      case 2: {
        T& v = F[2][at(x, 2, i, j, k)];
        v = upd(v, cdx[i], F[4][at(x, 4, i, j, k)], F[4][at(x, 4, i - 1, j, k)], cdy[j], F[3][at(x, 3, i, j, k)],
                F[3][at(x, 3, i, j - 1, k)]);
        break;
      }
      case 3: {
        T& v = F[3][at(x, 3, i, j, k)];
        v = upd(v, cdz[k], F[1][at(x, 1, i, j, k + 1)], F[1][at(x, 1, i, j, k)], cdy[j], F[2][at(x, 2, i, j + 1, k)],
                F[2][at(x, 2, i, j, k)]);
        break;
      }
      case 4: {
        T& v = F[4][at(x, 4, i, j, k)];
        v = upd(v, cdx[i], F[2][at(x, 2, i + 1, j, k)], F[2][at(x, 2, i, j, k)], cdz[k], F[0][at(x, 0, i, j, k + 1)],
                F[0][at(x, 0, i, j, k)]);
        break;
      }
      default: {
        T& v = F[5][at(x, 5, i, j, k)];
        v = upd(v, cdy[j], F[0][at(x, 0, i, j + 1, k)], F[0][at(x, 0, i, j, k)], cdx[i], F[1][at(x, 1, i + 1, j, k)],
                F[1][at(x, 1, i, j, k)]);
        break;
      }
    }
  }
}

// Dual spacing at node index i (fields.hpp:86-93): half-sum of the adjacent
// cells, halved at the domain ends.
__device__ __forceinline__ double dual(const double* d, int n, int i) {
  if (i == 0) return 0.5 * d[0];
  if (i == n) return 0.5 * d[n - 1];
  return 0.5 * (d[i - 1] + d[i]);
}

constexpr int kDenseEnergyBlocks = 296;

// total_energy (fields.hpp:116-146): sum_E V*E^2 + sum_H V*Hprev*Hnow in
// double. Fixed grid and a fixed per-block tree, so the sum is deterministic
// (its order differs from the reference's serial loop).
template <class T>
__global__ void __launch_bounds__(256) k_energy_dense(HostFields<T> f, const T* p3, const T* p4, const T* p5,
                                                      HostExt x, const double* dx, const double* dy,
                                                      const double* dz, int nx, int ny, int nz,
                                                      double* partial) {
  const int c = blockIdx.y;
  const T* now = f.f[c];
  const T* prev = c == 3 ? p3 : (c == 4 ? p4 : (c == 5 ? p5 : now));
  const int ex = x.e[c][0], ey = x.e[c][1], ez = x.e[c][2];
  const int axis = c % 3;
  const bool node[3] = {c < 3 ? axis != 0 : axis == 0, c < 3 ? axis != 1 : axis == 1,
                        c < 3 ? axis != 2 : axis == 2};
  const long long n = (long long)ex * ey * ez;
  double acc = 0.0;
  for (long long t = blockIdx.x * 256LL + threadIdx.x; t < n; t += (long long)gridDim.x * 256) {
    const int i = (int)(t % ex), j = (int)((t / ex) % ey), k = (int)(t / ((long long)ex * ey));
    const double vx = node[0] ? dual(dx, nx, i) : dx[i];
    const double vy = node[1] ? dual(dy, ny, j) : dy[j];
    const double vz = node[2] ? dual(dz, nz, k) : dz[k];
    acc += vx * vy * vz * (double)prev[t] * (double)now[t];
  }
  __shared__ double red[256];
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[c * gridDim.x + blockIdx.x] = red[0];
}

__global__ void k_energy_sum(const double* partial, int n, double* out) {
  double s = 0.0;
  for (int q = 0; q < n; ++q) s += partial[q];
  *out = s;
}

}  // namespace

template <class T>
cudaError_t launch_host_box(const HostFields<T>& f, const HostExt& x, int op, int comp, const HostBox& b,
                            cudaStream_t st) {
  const long long n = (long long)(b.xhi - b.xlo) * (b.yhi - b.ylo) * (b.zhi - b.zlo);
  if (n <= 0) return cudaSuccess;
  const int blocks = (int)((n + 255) / 256 < 148 * 16 ? (n + 255) / 256 : 148 * 16);
  k_box<T><<<blocks, 256, 0, st>>>(f, x, op, comp, b);
  return cudaGetLastError();
}

template <class T>
cudaError_t launch_host_energy(const HostFields<T>& f, const T* const* prev_h, const HostExt& x,
                               const double* dxyz, int nx, int ny, int nz, double* scratch, cudaStream_t st) {
  k_energy_dense<T><<<dim3(kDenseEnergyBlocks, 6), 256, 0, st>>>(f, prev_h[0], prev_h[1], prev_h[2], x, dxyz,
                                                             dxyz + nx, dxyz + nx + ny, nx, ny, nz, scratch);
  k_energy_sum<<<1, 1, 0, st>>>(scratch, 6 * kDenseEnergyBlocks, scratch + 6 * kDenseEnergyBlocks);
  return cudaGetLastError();
}

int host_energy_scratch_doubles() { return 6 * kDenseEnergyBlocks + 1; }

template cudaError_t launch_host_box<float>(const HostFields<float>&, const HostExt&, int, int, const HostBox&,
                                            cudaStream_t);
template cudaError_t launch_host_box<double>(const HostFields<double>&, const HostExt&, int, int, const HostBox&,
                                             cudaStream_t);
template cudaError_t launch_host_energy<float>(const HostFields<float>&, const float* const*, const HostExt&,
                                               const double*, int, int, int, double*, cudaStream_t);
template cudaError_t launch_host_energy<double>(const HostFields<double>&, const double* const*, const HostExt&,
                                                const double*, int, int, int, double*, cudaStream_t);

}  // namespace yb
