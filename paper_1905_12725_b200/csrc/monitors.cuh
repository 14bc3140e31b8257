// monitors.cuh — residual-monitor kernels (monitors.cu), P:270-290 / P:327-330.
#pragma once
#include "cg.cuh"

int monitor_blocks();
// (curl v)_j = e_jkl i xi_k v_l of one tensor row (3 spectral fields, layout of SpecGeom), in place
cudaError_t launch_curl3(const SpecGeom& g, cplx* v, cudaStream_t s);
// eta = curl curl eps of a symmetric field (6 Voigt spectral fields xx,yy,zz,yz,xz,xy), in place
cudaError_t launch_curlcurl6(const SpecGeom& g, cplx* v, cudaStream_t s);
// per-block max |x| over n doubles -> partials[monitor_blocks()]
cudaError_t launch_maxabs(const double* x, long long n, double* partials, cudaStream_t s);
// per-block sum of n doubles -> partials[monitor_blocks()]
cudaError_t launch_sum(const double* x, long long n, double* partials, cudaStream_t s);
// per-block sum_xi w |v|^2 over nf spectral fields -> partials[monitor_blocks()]
cudaError_t launch_specnorm2(const SpecGeom& g, const cplx* v, int nf, double* partials, cudaStream_t s);
