// monitors.cu — pointwise spectral kernels and reductions of the residual monitors (P:270-290,
// P:327-330).  The transforms around them are the column / X passes of passes.cu.
#include "monitors.cuh"

namespace {

constexpr int MB = 256;
static int mnb() { return 4 * num_sms(); }  // monitor grid: 4 CTAs per SM

DBF_DEV int eps3(int i, int j, int k) {  // Levi-Civita symbol
  return (i == j || j == k || i == k) ? 0 : (((j - i + 3) % 3) == 1 ? 1 : -1);
}

// rows of a tensor field, one row (3 fields v_l) at a time: (curl v)_j = e_jkl i xi_k v_l, in place
__global__ void __launch_bounds__(MB) k_curl3(SpecGeom g, cplx* __restrict__ v) {
  for (long long i = (long long)blockIdx.x * MB + threadIdx.x; i < g.Hs; i += (long long)gridDim.x * MB) {
    const Pt p = point(g, i);
    const double xi[3] = {p.xx, p.xy, p.xz};
    cplx a[3], c[3];
#pragma unroll
    for (int l = 0; l < 3; ++l) a[l] = v[l * g.Hs + i];
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      double re = 0.0, im = 0.0;  // sum_kl e_jkl xi_k a_l, then times i
#pragma unroll
      for (int k = 0; k < 3; ++k)
#pragma unroll
        for (int l = 0; l < 3; ++l) {
          const int e = eps3(j, k, l);
          if (e) {
            re += e * xi[k] * a[l].x;
            im += e * xi[k] * a[l].y;
          }
        }
      c[j] = make_double2(-im, re);
    }
#pragma unroll
    for (int j = 0; j < 3; ++j) v[j * g.Hs + i] = c[j];
  }
}

// incompatibility of a symmetric field (Voigt xx,yy,zz,yz,xz,xy):
// eta_ij = e_ikl e_jmn d_k d_m eps_ln  ->  -e_ikl e_jmn xi_k xi_m eps_ln, in place
__global__ void __launch_bounds__(MB) k_curlcurl6(SpecGeom g, cplx* __restrict__ v) {
  const int vo[3][3] = {{0, 5, 4}, {5, 1, 3}, {4, 3, 2}};
  for (long long i = (long long)blockIdx.x * MB + threadIdx.x; i < g.Hs; i += (long long)gridDim.x * MB) {
    const Pt p = point(g, i);
    const double xi[3] = {p.xx, p.xy, p.xz};
    cplx e6[6];
#pragma unroll
    for (int a = 0; a < 6; ++a) e6[a] = v[a * g.Hs + i];
    cplx T[3][3];  // T_in = sum_kl e_ikl xi_k eps_ln
#pragma unroll
    for (int ii = 0; ii < 3; ++ii)
#pragma unroll
      for (int n = 0; n < 3; ++n) {
        double re = 0.0, im = 0.0;
#pragma unroll
        for (int k = 0; k < 3; ++k)
#pragma unroll
          for (int l = 0; l < 3; ++l) {
            const int e = eps3(ii, k, l);
            if (e) {
              re += e * xi[k] * e6[vo[l][n]].x;
              im += e * xi[k] * e6[vo[l][n]].y;
            }
          }
        T[ii][n] = make_double2(re, im);
      }
    const int I6[6] = {0, 1, 2, 1, 0, 0}, J6[6] = {0, 1, 2, 2, 2, 1};
#pragma unroll
    for (int a = 0; a < 6; ++a) {
      const int ii = I6[a], j = J6[a];
      double re = 0.0, im = 0.0;  // -sum_mn e_jmn xi_m T_in
#pragma unroll
      for (int m = 0; m < 3; ++m)
#pragma unroll
        for (int n = 0; n < 3; ++n) {
          const int e = eps3(j, m, n);
          if (e) {
            re -= e * xi[m] * T[ii][n].x;
            im -= e * xi[m] * T[ii][n].y;
          }
        }
      v[a * g.Hs + i] = make_double2(re, im);
    }
  }
}

// per-block max |x|
__global__ void __launch_bounds__(MB) k_maxabs(const double* __restrict__ x, long long n, double* partials) {
  double m = 0.0;
  for (long long i = (long long)blockIdx.x * MB + threadIdx.x; i < n; i += (long long)gridDim.x * MB) m = fmax(m, fabs(x[i]));
  __shared__ double red[MB / 32];
  m = warp_max(m);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < MB / 32; ++w) s = fmax(s, red[w]);
    partials[blockIdx.x] = s;
  }
}

// per-block sum of x
__global__ void __launch_bounds__(MB) k_sum(const double* __restrict__ x, long long n, double* partials) {
  double m = 0.0;
  for (long long i = (long long)blockIdx.x * MB + threadIdx.x; i < n; i += (long long)gridDim.x * MB) m += x[i];
  __shared__ double red[MB / 32];
  m = warp_sum(m);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < MB / 32; ++w) s += red[w];
    partials[blockIdx.x] = s;
  }
}

// per-block sum_xi w |v(xi)|^2 over nf spectral fields (Parseval with the half spectrum, R6)
__global__ void __launch_bounds__(MB) k_specnorm2(SpecGeom g, const cplx* __restrict__ v, int nf, double* partials) {
  double s = 0.0;
  for (long long i = (long long)blockIdx.x * MB + threadIdx.x; i < g.Hs; i += (long long)gridDim.x * MB) {
    const int kx = (int)(i % g.n1h);
    const double w = (kx + g.kx0 == 0 || 2 * (kx + g.kx0) == g.n1) ? 1.0 : 2.0;
    for (int f = 0; f < nf; ++f) {
      const cplx a = v[f * g.Hs + i];
      s += w * (a.x * a.x + a.y * a.y);
    }
  }
  __shared__ double red[MB / 32];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < MB / 32; ++w) t += red[w];
    partials[blockIdx.x] = t;
  }
}

}  // namespace

int monitor_blocks() { return mnb(); }

cudaError_t launch_curl3(const SpecGeom& g, cplx* v, cudaStream_t s) {
  k_curl3<<<mnb(), MB, 0, s>>>(g, v);
  return cudaGetLastError();
}
cudaError_t launch_curlcurl6(const SpecGeom& g, cplx* v, cudaStream_t s) {
  k_curlcurl6<<<mnb(), MB, 0, s>>>(g, v);
  return cudaGetLastError();
}
cudaError_t launch_maxabs(const double* x, long long n, double* partials, cudaStream_t s) {
  k_maxabs<<<mnb(), MB, 0, s>>>(x, n, partials);
  return cudaGetLastError();
}
cudaError_t launch_sum(const double* x, long long n, double* partials, cudaStream_t s) {
  k_sum<<<mnb(), MB, 0, s>>>(x, n, partials);
  return cudaGetLastError();
}
cudaError_t launch_specnorm2(const SpecGeom& g, const cplx* v, int nf, double* partials, cudaStream_t s) {
  k_specnorm2<<<mnb(), MB, 0, s>>>(g, v, nf, partials);
  return cudaGetLastError();
}
