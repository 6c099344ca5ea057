// small_kernels.cu -- see small_kernels.cuh.
#include <algorithm>

#include "small_kernels.cuh"

namespace chfsi {

namespace {

__global__ void hemv_kernel(int64_t n, int64_t nloc, const double2* __restrict__ Hp, const void* const* hpp,
                            int64_t ldh, const double2* __restrict__ v, double2* __restrict__ w) {
  const int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= nloc) return;
  if (hpp) Hp = static_cast<const double2*>(*hpp);  // H through a device slot (the captured Lanczos graph)
  const double2* h = Hp + r * ldh;
  double sr0 = 0, si0 = 0, sr1 = 0, si1 = 0;
  int64_t q = lane;
  for (; q + 32 < n; q += 64) {
    const double2 a = __ldcs(h + q), b = __ldcs(h + q + 32);
    const double2 x = __ldg(v + q), y = __ldg(v + q + 32);
    sr0 += a.x * x.x + a.y * x.y;
    si0 += a.x * x.y - a.y * x.x;
    sr1 += b.x * y.x + b.y * y.y;
    si1 += b.x * y.y - b.y * y.x;
  }
  if (q < n) {
    const double2 a = __ldcs(h + q);
    const double2 x = __ldg(v + q);
    sr0 += a.x * x.x + a.y * x.y;
    si0 += a.x * x.y - a.y * x.x;
  }
  double sr = warp_sum(sr0 + sr1), si = warp_sum(si0 + si1);
  if (lane == 0) w[r] = make_double2(sr, si);
}

// K entry q of chunk c = q / chunk lands at c * ldk + q % chunk (ldk >= chunk; the gaps are zero)
__global__ void h3_plane_kernel(int64_t n, int64_t nloc, const double2* __restrict__ Hp, int64_t ldh,
                                double* __restrict__ H3, int64_t ld3, int64_t chunk, int64_t ldk) {
  const int64_t nchunks = (n + chunk - 1) / chunk;
  for (int64_t r = blockIdx.y; r < nloc; r += gridDim.y)
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nchunks * ldk;
         i += (int64_t)gridDim.x * blockDim.x) {
      const int64_t c = i / ldk, o = i - c * ldk, q = c * chunk + o;
      double v = 0.0;
      if (o < chunk && q < n) {
        const double2 h = __ldcs(Hp + r * ldh + q);
        v = h.x - h.y;
      }
      H3[r * ld3 + i] = v;
    }
}

__global__ void pack_y3_kernel(int64_t rows, int64_t cols, const double2* __restrict__ X, int64_t ldx,
                               double* __restrict__ dst, int64_t cs, int64_t y3_off) {
  for (int64_t j = blockIdx.y; j < cols; j += gridDim.y) {
    double* col = dst + j * cs;
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x) {
      const double2 x = X[j * ldx + r];
      reinterpret_cast<double2*>(col)[r] = x;
      col[y3_off + r] = x.x + x.y;
    }
  }
}

template <int NT>
__device__ double block_sum(double v) {
  __shared__ double red[NT / 32];
  v = warp_sum(v);
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) red[wid] = v;
  __syncthreads();
  double s = 0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NT / 32; ++i) s += red[i];
  }
  return s;
}

constexpr int kRedThreads = 256;

__global__ void colnorm2_kernel(int64_t rows, const double2* __restrict__ X, int64_t ldx, double* out) {
  const double2* x = X + (int64_t)blockIdx.x * ldx;
  double s = 0;
  for (int64_t r = threadIdx.x; r < rows; r += kRedThreads) {
    const double2 a = x[r];
    s += a.x * a.x + a.y * a.y;
  }
  s = block_sum<kRedThreads>(s);
  if (threadIdx.x == 0) out[blockIdx.x] = s;
}

__global__ void resid2_kernel(int64_t rows, const double2* __restrict__ HY, int64_t ld1, const double2* __restrict__ Y,
                              int64_t ld2, const double* __restrict__ mu, double* out) {
  const double2* hy = HY + (int64_t)blockIdx.x * ld1;
  const double2* y = Y + (int64_t)blockIdx.x * ld2;
  const double m = mu[blockIdx.x];
  double s = 0;
  for (int64_t r = threadIdx.x; r < rows; r += kRedThreads) {
    const double2 a = hy[r], b = y[r];
    const double dr = a.x - m * b.x, di = a.y - m * b.y;
    s += dr * dr + di * di;
  }
  s = block_sum<kRedThreads>(s);
  if (threadIdx.x == 0) out[blockIdx.x] = s;
}

__global__ void hermitize_kernel(int64_t k, double2* G, int64_t ldg) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (int64_t j = blockIdx.y; j < k; j += gridDim.y) {
    if (i > j) continue;
    const double2 a = G[j * ldg + i], b = G[i * ldg + j];
    if (i == j) {
      G[j * ldg + i] = make_double2(a.x, 0.0);
      continue;
    }
    // upper (i,j) = (a + conj(b))/2, lower (j,i) = conj(upper)
    const double2 u = make_double2(0.5 * (a.x + b.x), 0.5 * (a.y - b.y));
    G[j * ldg + i] = u;
    G[i * ldg + j] = make_double2(u.x, -u.y);
  }
}

__global__ void col_gather_kernel(int64_t rows, int64_t cols, const double2* __restrict__ src, int64_t lds,
                                  const int* __restrict__ idx, double2* __restrict__ dst, int64_t ldd) {
  for (int64_t j = blockIdx.y; j < cols; j += gridDim.y) {
    const double2* s = src + (int64_t)idx[j] * lds;
    double2* d = dst + j * ldd;
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x)
      d[r] = s[r];
  }
}

__global__ void col_phase_kernel(int64_t rows, int64_t cols, double2* Q, int64_t ldq, const double2* R, int64_t ldr) {
  for (int64_t j = blockIdx.y; j < cols; j += gridDim.y) {
    const double2 d = R[j * ldr + j];
    const double a = hypot(d.x, d.y);
    const double pr = a > 0 ? d.x / a : 1.0, pi = a > 0 ? d.y / a : 0.0;
    double2* q = Q + j * ldq;
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x) {
      const double2 x = q[r];
      q[r] = make_double2(x.x * pr - x.y * pi, x.x * pi + x.y * pr);
    }
  }
}

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

__global__ void random_block_kernel(int64_t rows, int64_t cols, int64_t row0, uint64_t seed, uint64_t stream_base,
                                    uint64_t stream_stride, double2* X, int64_t ldx) {
  for (int64_t j = blockIdx.y; j < cols; j += gridDim.y) {
    const uint64_t strm = stream_base | (stream_stride * (uint64_t)j);
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x) {
      const uint64_t g = (uint64_t)(row0 + r);
      const uint64_t h0 = splitmix64(seed ^ (strm << 40) ^ (2 * g));
      const uint64_t h1 = splitmix64(seed ^ (strm << 40) ^ (2 * g + 1));
      const double u0 = (double)(h0 >> 11) * (1.0 / 9007199254740992.0);
      const double u1 = (double)(h1 >> 11) * (1.0 / 9007199254740992.0);
      X[j * ldx + r] = make_double2(__dadd_rn(__dmul_rn(2.0, u0), -1.0), __dadd_rn(__dmul_rn(2.0, u1), -1.0));
    }
  }
}

__global__ void scale_kernel(int64_t rows, double2* x, double s) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x) {
    const double2 a = x[r];
    x[r] = make_double2(a.x * s, a.y * s);
  }
}

template <typename D>
__global__ void scale_rnorm_kernel(int64_t rows, D* x, const double* nrm2) {
  const double s = 1.0 / sqrt(*nrm2);
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x) {
    if constexpr (sizeof(D) == 16) {
      const double2 a = reinterpret_cast<const double2*>(x)[r];
      reinterpret_cast<double2*>(x)[r] = make_double2(a.x * s, a.y * s);
    } else {
      reinterpret_cast<double*>(x)[r] *= s;
    }
  }
}

__global__ void store_ptr_kernel(const void** slot, const void* ptr) { *slot = ptr; }

// Lanczos step on the device (no host round trip): beta = sqrt(||w||^2), v_next = w / beta (nullable),
// alpha = Re(coef_j) (nullable); beta and alpha land in the step's slots of the device arrays
template <typename D>
__global__ void lanczos_next_kernel(int64_t rows, const D* __restrict__ w, D* __restrict__ vn, const double* nrm2,
                                    const D* coef_j, double* beta_out, double* alpha_out) {
  const double beta = sqrt(*nrm2);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *beta_out = beta;
    if (alpha_out) {
      if constexpr (sizeof(D) == 16) {
        *alpha_out = reinterpret_cast<const double2*>(coef_j)->x;
      } else {
        *alpha_out = *reinterpret_cast<const double*>(coef_j);
      }
    }
  }
  if (!vn) return;
  const double s = 1.0 / beta;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x) {
    if constexpr (sizeof(D) == 16) {
      const double2 a = reinterpret_cast<const double2*>(w)[r];
      reinterpret_cast<double2*>(vn)[r] = make_double2(a.x * s, a.y * s);
    } else {
      reinterpret_cast<double*>(vn)[r] = reinterpret_cast<const double*>(w)[r] * s;
    }
  }
}

__global__ void orth_err_kernel(int64_t k, const double2* G, int64_t ldg, unsigned long long* out) {
  double m = 0;
  for (int64_t j = blockIdx.y; j < k; j += gridDim.y)
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < k; i += (int64_t)gridDim.x * blockDim.x) {
      const double2 a = G[j * ldg + i];
      const double e = hypot(a.x - (i == j ? 1.0 : 0.0), a.y);
      m = fmax(m, e);
    }
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, __double_as_longlong(m));  // m >= 0: bit order == value order
}

// gridDim.y limit: the column-indexed kernels loop j += gridDim.y
inline unsigned ycap(int64_t cols) { return (unsigned)std::min<int64_t>(cols, 65535); }

inline unsigned grid1(int64_t rows, int threads) {
  int64_t b = (rows + threads - 1) / threads;
  return (unsigned)(b < 1 ? 1 : (b > 1024 ? 1024 : b));
}

}  // namespace

cudaError_t launch_hemv(int64_t n, int64_t nloc, const double2* Hp, int64_t ldh, const double2* v, double2* w,
                        cudaStream_t st, const void* const* hpp) {
  const int warps = 8;
  hemv_kernel<<<(unsigned)((nloc + warps - 1) / warps), warps * 32, 0, st>>>(n, nloc, Hp, hpp, ldh, v, w);
  return cudaGetLastError();
}

cudaError_t launch_colnorm2(int64_t rows, int64_t cols, const double2* X, int64_t ldx, double* out, cudaStream_t st) {
  if (cols <= 0) return cudaSuccess;
  colnorm2_kernel<<<(unsigned)cols, kRedThreads, 0, st>>>(rows, X, ldx, out);
  return cudaGetLastError();
}

cudaError_t launch_resid2(int64_t rows, int64_t cols, const double2* HY, int64_t ld1, const double2* Y, int64_t ld2,
                          const double* mu, double* out, cudaStream_t st) {
  if (cols <= 0) return cudaSuccess;
  resid2_kernel<<<(unsigned)cols, kRedThreads, 0, st>>>(rows, HY, ld1, Y, ld2, mu, out);
  return cudaGetLastError();
}

cudaError_t launch_hermitize(int64_t k, double2* G, int64_t ldg, cudaStream_t st) {
  if (k <= 0) return cudaSuccess;
  dim3 grid((unsigned)((k + 127) / 128), (unsigned)std::min<int64_t>(k, 65535));
  hermitize_kernel<<<grid, 128, 0, st>>>(k, G, ldg);
  return cudaGetLastError();
}

cudaError_t launch_col_gather(int64_t rows, int64_t cols, const double2* src, int64_t lds, const int* idx,
                              double2* dst, int64_t ldd, cudaStream_t st) {
  if (cols <= 0 || rows <= 0) return cudaSuccess;
  dim3 grid(grid1(rows, 256) > 64 ? 64 : grid1(rows, 256), ycap(cols));
  col_gather_kernel<<<grid, 256, 0, st>>>(rows, cols, src, lds, idx, dst, ldd);
  return cudaGetLastError();
}

cudaError_t launch_col_phase(int64_t rows, int64_t cols, double2* Q, int64_t ldq, const double2* R, int64_t ldr,
                             cudaStream_t st) {
  if (cols <= 0 || rows <= 0) return cudaSuccess;
  dim3 grid(grid1(rows, 256) > 64 ? 64 : grid1(rows, 256), ycap(cols));
  col_phase_kernel<<<grid, 256, 0, st>>>(rows, cols, Q, ldq, R, ldr);
  return cudaGetLastError();
}

cudaError_t launch_random_block(int64_t rows, int64_t cols, int64_t row0, uint64_t seed, uint64_t stream_base,
                                uint64_t stream_stride, double2* X, int64_t ldx, cudaStream_t st) {
  if (cols <= 0 || rows <= 0) return cudaSuccess;
  dim3 grid(grid1(rows, 256) > 64 ? 64 : grid1(rows, 256), ycap(cols));
  random_block_kernel<<<grid, 256, 0, st>>>(rows, cols, row0, seed, stream_base, stream_stride, X, ldx);
  return cudaGetLastError();
}

cudaError_t launch_scale(int64_t rows, double2* x, double s, cudaStream_t st) {
  scale_kernel<<<grid1(rows, 256), 256, 0, st>>>(rows, x, s);
  return cudaGetLastError();
}

cudaError_t launch_orth_err(int64_t k, const double2* G, int64_t ldg, double* out, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(out, 0, sizeof(double), st);
  if (e != cudaSuccess) return e;
  dim3 grid((unsigned)((k + 255) / 256), ycap(k));
  orth_err_kernel<<<grid, 256, 0, st>>>(k, G, ldg, reinterpret_cast<unsigned long long*>(out));
  return cudaGetLastError();
}

// ================================================================================================
// real-symmetric counterparts
namespace {

__global__ void hemv_real_kernel(int64_t n, int64_t nloc, const double* __restrict__ Hp, const void* const* hpp,
                                 int64_t ldh, const double* __restrict__ v, double* __restrict__ w) {
  const int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= nloc) return;
  if (hpp) Hp = static_cast<const double*>(*hpp);
  const double* h = Hp + r * ldh;
  double s0 = 0, s1 = 0;
  int64_t q = lane;
  for (; q + 32 < n; q += 64) {
    s0 += __ldcs(h + q) * __ldg(v + q);
    s1 += __ldcs(h + q + 32) * __ldg(v + q + 32);
  }
  if (q < n) s0 += __ldcs(h + q) * __ldg(v + q);
  const double s = warp_sum(s0 + s1);
  if (lane == 0) w[r] = s;
}

__global__ void colnorm2_real_kernel(int64_t rows, const double* __restrict__ X, int64_t ldx, double* out) {
  const double* x = X + (int64_t)blockIdx.x * ldx;
  double s = 0;
  for (int64_t r = threadIdx.x; r < rows; r += kRedThreads) s += x[r] * x[r];
  s = block_sum<kRedThreads>(s);
  if (threadIdx.x == 0) out[blockIdx.x] = s;
}

__global__ void resid2_real_kernel(int64_t rows, const double* __restrict__ HY, int64_t ld1,
                                   const double* __restrict__ Y, int64_t ld2, const double* __restrict__ mu,
                                   double* out) {
  const double* hy = HY + (int64_t)blockIdx.x * ld1;
  const double* y = Y + (int64_t)blockIdx.x * ld2;
  const double m = mu[blockIdx.x];
  double s = 0;
  for (int64_t r = threadIdx.x; r < rows; r += kRedThreads) {
    const double d = hy[r] - m * y[r];
    s += d * d;
  }
  s = block_sum<kRedThreads>(s);
  if (threadIdx.x == 0) out[blockIdx.x] = s;
}

__global__ void symmetrize_kernel(int64_t k, double* G, int64_t ldg) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (int64_t j = blockIdx.y; j < k; j += gridDim.y) {
    if (i >= j) continue;
    const double u = 0.5 * (G[j * ldg + i] + G[i * ldg + j]);
    G[j * ldg + i] = u;
    G[i * ldg + j] = u;
  }
}

__global__ void col_gather_real_kernel(int64_t rows, int64_t cols, const double* __restrict__ src, int64_t lds,
                                       const int* __restrict__ idx, double* __restrict__ dst, int64_t ldd) {
  for (int64_t j = blockIdx.y; j < cols; j += gridDim.y) {
    const double* s = src + (int64_t)idx[j] * lds;
    double* d = dst + j * ldd;
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x)
      d[r] = s[r];
  }
}

__global__ void col_sign_kernel(int64_t rows, int64_t cols, double* Q, int64_t ldq, const double* R, int64_t ldr) {
  for (int64_t j = blockIdx.y; j < cols; j += gridDim.y) {
    const double sgn = R[j * ldr + j] < 0 ? -1.0 : 1.0;
    double* q = Q + j * ldq;
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x)
      q[r] *= sgn;
  }
}

__global__ void random_block_real_kernel(int64_t rows, int64_t cols, int64_t row0, uint64_t seed,
                                         uint64_t stream_base, uint64_t stream_stride, double* X, int64_t ldx) {
  for (int64_t j = blockIdx.y; j < cols; j += gridDim.y) {
    const uint64_t strm = stream_base | (stream_stride * (uint64_t)j);
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x) {
      const uint64_t g = (uint64_t)(row0 + r);
      const uint64_t h0 = splitmix64(seed ^ (strm << 40) ^ (2 * g));
      const double u0 = (double)(h0 >> 11) * (1.0 / 9007199254740992.0);
      X[j * ldx + r] = __dadd_rn(__dmul_rn(2.0, u0), -1.0);
    }
  }
}

__global__ void scale_real_kernel(int64_t rows, double* x, double s) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x)
    x[r] *= s;
}

__global__ void orth_err_real_kernel(int64_t k, const double* G, int64_t ldg, unsigned long long* out) {
  double m = 0;
  for (int64_t j = blockIdx.y; j < k; j += gridDim.y)
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < k; i += (int64_t)gridDim.x * blockDim.x)
      m = fmax(m, fabs(G[j * ldg + i] - (i == j ? 1.0 : 0.0)));
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, __double_as_longlong(m));
}

}  // namespace

cudaError_t launch_hemv(int64_t n, int64_t nloc, const double* Hp, int64_t ldh, const double* v, double* w,
                        cudaStream_t st, const void* const* hpp) {
  const int warps = 8;
  hemv_real_kernel<<<(unsigned)((nloc + warps - 1) / warps), warps * 32, 0, st>>>(n, nloc, Hp, hpp, ldh, v, w);
  return cudaGetLastError();
}
cudaError_t launch_colnorm2(int64_t rows, int64_t cols, const double* X, int64_t ldx, double* out, cudaStream_t st) {
  if (cols <= 0) return cudaSuccess;
  colnorm2_real_kernel<<<(unsigned)cols, kRedThreads, 0, st>>>(rows, X, ldx, out);
  return cudaGetLastError();
}
cudaError_t launch_resid2(int64_t rows, int64_t cols, const double* HY, int64_t ld1, const double* Y, int64_t ld2,
                          const double* mu, double* out, cudaStream_t st) {
  if (cols <= 0) return cudaSuccess;
  resid2_real_kernel<<<(unsigned)cols, kRedThreads, 0, st>>>(rows, HY, ld1, Y, ld2, mu, out);
  return cudaGetLastError();
}
cudaError_t launch_hermitize(int64_t k, double* G, int64_t ldg, cudaStream_t st) {
  if (k <= 0) return cudaSuccess;
  dim3 grid((unsigned)((k + 127) / 128), (unsigned)std::min<int64_t>(k, 65535));
  symmetrize_kernel<<<grid, 128, 0, st>>>(k, G, ldg);
  return cudaGetLastError();
}
cudaError_t launch_col_gather(int64_t rows, int64_t cols, const double* src, int64_t lds, const int* idx, double* dst,
                              int64_t ldd, cudaStream_t st) {
  if (cols <= 0 || rows <= 0) return cudaSuccess;
  dim3 grid(grid1(rows, 256) > 64 ? 64 : grid1(rows, 256), ycap(cols));
  col_gather_real_kernel<<<grid, 256, 0, st>>>(rows, cols, src, lds, idx, dst, ldd);
  return cudaGetLastError();
}
cudaError_t launch_col_phase(int64_t rows, int64_t cols, double* Q, int64_t ldq, const double* R, int64_t ldr,
                             cudaStream_t st) {
  if (cols <= 0 || rows <= 0) return cudaSuccess;
  dim3 grid(grid1(rows, 256) > 64 ? 64 : grid1(rows, 256), ycap(cols));
  col_sign_kernel<<<grid, 256, 0, st>>>(rows, cols, Q, ldq, R, ldr);
  return cudaGetLastError();
}
cudaError_t launch_random_block(int64_t rows, int64_t cols, int64_t row0, uint64_t seed, uint64_t stream_base,
                                uint64_t stream_stride, double* X, int64_t ldx, cudaStream_t st) {
  if (cols <= 0 || rows <= 0) return cudaSuccess;
  dim3 grid(grid1(rows, 256) > 64 ? 64 : grid1(rows, 256), ycap(cols));
  random_block_real_kernel<<<grid, 256, 0, st>>>(rows, cols, row0, seed, stream_base, stream_stride, X, ldx);
  return cudaGetLastError();
}
cudaError_t launch_scale(int64_t rows, double* x, double s, cudaStream_t st) {
  scale_real_kernel<<<grid1(rows, 256), 256, 0, st>>>(rows, x, s);
  return cudaGetLastError();
}
cudaError_t launch_orth_err(int64_t k, const double* G, int64_t ldg, double* out, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(out, 0, sizeof(double), st);
  if (e != cudaSuccess) return e;
  dim3 grid((unsigned)((k + 255) / 256), ycap(k));
  orth_err_real_kernel<<<grid, 256, 0, st>>>(k, G, ldg, reinterpret_cast<unsigned long long*>(out));
  return cudaGetLastError();
}

cudaError_t launch_h3_plane(int64_t n, int64_t nloc, const double2* Hp, int64_t ldh, double* H3, int64_t ld3,
                            int64_t chunk, int64_t ldk, cudaStream_t st) {
  if (n <= 0 || nloc <= 0) return cudaSuccess;
  const int64_t len = (n + chunk - 1) / chunk * ldk;
  const unsigned bx = (unsigned)std::min<int64_t>((len + 255) / 256, 16);
  h3_plane_kernel<<<dim3(bx, (unsigned)std::min<int64_t>(nloc, 65535)), 256, 0, st>>>(n, nloc, Hp, ldh, H3, ld3, chunk, ldk);
  return cudaGetLastError();
}

cudaError_t launch_pack_y3(int64_t rows, int64_t cols, const double2* X, int64_t ldx, double* dst, int64_t cs,
                           int64_t y3_off, cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return cudaSuccess;
  const unsigned bx = (unsigned)std::min<int64_t>((rows + 255) / 256, 64);
  pack_y3_kernel<<<dim3(bx, ycap(cols)), 256, 0, st>>>(rows, cols, X, ldx, dst, cs, y3_off);
  return cudaGetLastError();
}

cudaError_t launch_lanczos_next(int64_t rows, const double2* w, double2* vn, const double* nrm2, const double2* coef_j,
                                double* beta_out, double* alpha_out, cudaStream_t st) {
  lanczos_next_kernel<double2><<<grid1(rows, 256), 256, 0, st>>>(rows, w, vn, nrm2, coef_j, beta_out, alpha_out);
  return cudaGetLastError();
}

cudaError_t launch_lanczos_next(int64_t rows, const double* w, double* vn, const double* nrm2, const double* coef_j,
                                double* beta_out, double* alpha_out, cudaStream_t st) {
  lanczos_next_kernel<double><<<grid1(rows, 256), 256, 0, st>>>(rows, w, vn, nrm2, coef_j, beta_out, alpha_out);
  return cudaGetLastError();
}

cudaError_t launch_scale_rnorm(int64_t rows, double2* x, const double* nrm2, cudaStream_t st) {
  scale_rnorm_kernel<double2><<<grid1(rows, 256), 256, 0, st>>>(rows, x, nrm2);
  return cudaGetLastError();
}
cudaError_t launch_scale_rnorm(int64_t rows, double* x, const double* nrm2, cudaStream_t st) {
  scale_rnorm_kernel<double><<<grid1(rows, 256), 256, 0, st>>>(rows, x, nrm2);
  return cudaGetLastError();
}
cudaError_t launch_store_ptr(const void** slot, const void* ptr, cudaStream_t st) {
  store_ptr_kernel<<<1, 1, 0, st>>>(slot, ptr);
  return cudaGetLastError();
}

}  // namespace chfsi
