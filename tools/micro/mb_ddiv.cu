#include <cstdio>
__global__ void k(double* o, double a, double b, int n) {
  double x = a, y = b;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { x = y / x; y = x + 1.0; }
  long long t1 = clock64();
  float xf = (float)a, yf = (float)b;
  for (int i = 0; i < n; ++i) { xf = __fdiv_rn(yf, xf); yf = xf + 1.0f; }
  long long t2 = clock64();
  double z = a;
  for (int i = 0; i < n; ++i) { z = z + b; }
  long long t3 = clock64();
  double w = a;
  for (int i = 0; i < n; ++i) { w = __shfl_xor_sync(0xffffffff, w, 1) + b; }
  long long t4 = clock64();
  o[0] = x + xf + z + w; o[1] = (double)(t1 - t0) / n; o[2] = (double)(t2 - t1) / n; o[3] = (double)(t3 - t2) / n; o[4] = (double)(t4 - t3) / n;
}
int main() { double* d; cudaMalloc(&d, 64); k<<<1, 32>>>(d, 1.5, 2.5, 1000); double h[5]; cudaMemcpy(h, d, 40, cudaMemcpyDeviceToHost);
  printf("fp64 div+add chain %.1f cyc/iter, fp32 div+add %.1f, DADD %.1f, shfl64+DADD %.1f\n", h[1], h[2], h[3], h[4]); }
