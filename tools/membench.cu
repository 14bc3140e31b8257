// membench.cu — HBM copy throughput of the column-pass access patterns (tools only, not product).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o membench tools/membench.cu
// Patterns (complex128 elements; a "plane" is P rows of W elements, row pitch W):
//   contiguous   : flat copy
//   tile<KC>     : CTA copies KC columns x P rows (one plane, kx block), rows strided by W
// Each pattern reads NF fields and writes NF fields of the same layout.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

typedef double2 cplx;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s line %d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

__global__ void k_contig(const cplx* __restrict__ in, cplx* __restrict__ out, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    out[i] = __ldg(in + i);
}

// tile copy: tile t -> (plane, kb); thread layout: KC columns per row, 256/KC rows per pass
template <int KC>
__global__ void __launch_bounds__(256) k_tile(const cplx* __restrict__ in, cplx* __restrict__ out, int W, int P,
                                              int nplanes, int nkb, long long fs, int nf) {
  const int c = threadIdx.x % KC, r0 = threadIdx.x / KC;
  constexpr int RS = 256 / KC;
  const long long ntiles = (long long)nplanes * nkb * nf;
  for (long long t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int f = (int)(t / ((long long)nplanes * nkb));
    const long long pt = t % ((long long)nplanes * nkb);
    const int plane = (int)(pt / nkb), kb = (int)(pt % nkb);
    const long long base = f * fs + (long long)plane * P * W + kb * KC + c;
    cplx v[8];
    for (int r = r0; r < P; r += 8 * RS) {
#pragma unroll
      for (int s = 0; s < 8; ++s) {
        const int rr = r + s * RS;
        v[s] = rr < P ? __ldg(in + base + (long long)rr * W) : make_double2(0, 0);
      }
#pragma unroll
      for (int s = 0; s < 8; ++s) {
        const int rr = r + s * RS;
        if (rr < P) out[base + (long long)rr * W] = v[s];
      }
    }
  }
}

int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 256;
  const int nf = argc > 2 ? atoi(argv[2]) : 6;
  const int W = argc > 3 ? atoi(argv[3]) : n / 2 + 1, P = n, nplanes = n;
  printf("n=%d nf=%d pitch=%d\n", n, nf, W);
  const long long fs = (long long)W * P * nplanes;
  const long long tot = fs * nf;
  cplx *a, *b;
  CK(cudaMalloc(&a, tot * sizeof(cplx)));
  CK(cudaMalloc(&b, tot * sizeof(cplx)));
  CK(cudaMemset(a, 0, tot * sizeof(cplx)));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  auto run = [&](const char* name, auto launch) {
    for (int i = 0; i < 3; ++i) launch();
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    const int reps = 10;
    for (int i = 0; i < reps; ++i) launch();
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= reps;
    printf("%-28s %8.3f ms  %7.1f GB/s\n", name, ms, 2.0 * tot * sizeof(cplx) / ms / 1e6);
  };
  run("contiguous", [&] { k_contig<<<nsm * 8, 256>>>(a, b, tot); });
  const int nkb = (n / 2) / 8;
  for (int occ : {4, 8, 16, 32}) {
    char nm[64];
    snprintf(nm, 64, "tile8 grid=%dxSM", occ);
    run(nm, [&] { k_tile<8><<<nsm * occ, 256>>>(a, b, W, P, nplanes, nkb, fs, nf); });
  }
  for (int occ : {8, 16}) {
    char nm[64];
    snprintf(nm, 64, "tile16 grid=%dxSM", occ);
    run(nm, [&] { k_tile<16><<<nsm * occ, 256>>>(a, b, W, P, nplanes, (n / 2) / 16, fs, nf); });
    snprintf(nm, 64, "tile4 grid=%dxSM", occ);
    run(nm, [&] { k_tile<4><<<nsm * occ, 256>>>(a, b, W, P, nplanes, (n / 2) / 4, fs, nf); });
    snprintf(nm, 64, "tile32 grid=%dxSM", occ);
    run(nm, [&] { k_tile<32><<<nsm * occ, 256>>>(a, b, W, P, nplanes, (n / 2) / 32, fs, nf); });
  }
  return 0;
}
