// Accuracy of the f64 MUFU seeds (RCP64H, RSQ64H) and of the refinements
// used by the fast f64 dyad: max relative error over random inputs.
#include <cstdio>
#include <cmath>
#include <cuda_runtime.h>
__device__ double rcp_seed(double x) { double y; asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x)); return y; }
__device__ double rsq_seed(double x) { double y; asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x)); return y; }
__global__ void k(double* out, int n) {
  double m[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    unsigned long long s = 0x9E3779B97F4A7C15ull * (i + 1);
    s ^= s >> 29; s *= 0xBF58476D1CE4E5B9ull; s ^= s >> 32;
    const double x = ldexp(1.0 + (double)(s >> 11) * 0x1p-53, (int)(s % 41) - 30);
    const double rt = 1.0 / x, qt = 1.0 / sqrt(x);
    double y = rcp_seed(x);
    m[0] = fmax(m[0], fabs(y - rt) / rt);
    double e = fma(-x, y, 1.0);
    double y1 = fma(y, fma(e, e, e), y);  // cubic
    m[1] = fmax(m[1], fabs(y1 - rt) / rt);
    double y2 = fma(y, e, y); e = fma(-x, y2, 1.0); y2 = fma(y2, e, y2);  // two Newton steps
    m[2] = fmax(m[2], fabs(y2 - rt) / rt);
    double z = rsq_seed(x);
    m[3] = fmax(m[3], fabs(z - qt) / qt);
    double f = fma(-x, z * z, 1.0);
    double z1 = fma(z * f, fma(0.375, f, 0.5), z);  // Halley
    m[4] = fmax(m[4], fabs(z1 - qt) / qt);
    const double h = 0.5 * x; double z2 = z;
    for (int j = 0; j < 2; ++j) { const double g = fma(-h, z2 * z2, 0.5); z2 = fma(z2, g, z2); }
    m[5] = fmax(m[5], fabs(z2 - qt) / qt);
    double z3 = z; { const double g = fma(-h, z3 * z3, 0.5); z3 = fma(z3, g, z3); }
    m[6] = fmax(m[6], fabs(z3 - qt) / qt);
  }
  for (int j = 0; j < 8; ++j) atomicMax((unsigned long long*)&out[j], (unsigned long long)__double_as_longlong(m[j]));
}
int main() {
  double* d; cudaMalloc(&d, 64); cudaMemset(d, 0, 64);
  k<<<592, 256>>>(d, 1 << 26);
  double h[8]; cudaMemcpy(h, d, 64, cudaMemcpyDeviceToHost);
  printf("rcp seed %.3e cubic %.3e newton2 %.3e | rsqrt seed %.3e halley %.3e newton2 %.3e newton1 %.3e\n", h[0], h[1], h[2], h[3], h[4], h[5], h[6]);
  return cudaDeviceSynchronize() != cudaSuccess;
}
