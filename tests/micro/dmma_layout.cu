// Verifies the assumed f64 mma.sync fragment layouts (m16n8k4) against a host matmul.
#include <cstdio>
#include <cmath>
#include <cuda_runtime.h>

__global__ void k(const double* A, const double* B, double* D) {
  const int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
  double a0 = A[g * 4 + t], a1 = A[(g + 8) * 4 + t];  // A 16x4 row-major
  double b0 = B[t * 8 + g];                            // B 4x8: (k=t, n=g)
  double c0 = 0, c1 = 0, c2 = 0, c3 = 0;
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
               : "+d"(c0), "+d"(c1), "+d"(c2), "+d"(c3) : "d"(a0), "d"(a1), "d"(b0));
  D[g * 8 + 2 * t] = c0;
  D[g * 8 + 2 * t + 1] = c1;
  D[(g + 8) * 8 + 2 * t] = c2;
  D[(g + 8) * 8 + 2 * t + 1] = c3;
}

int main() {
  double hA[64], hB[32], hD[128], ref[128];
  for (int i = 0; i < 64; ++i) hA[i] = std::sin(1.0 + i);
  for (int i = 0; i < 32; ++i) hB[i] = std::cos(2.0 + 3 * i);
  for (int r = 0; r < 16; ++r)
    for (int c = 0; c < 8; ++c) {
      double s = 0;
      for (int q = 0; q < 4; ++q) s += hA[r * 4 + q] * hB[q * 8 + c];
      ref[r * 8 + c] = s;
    }
  double *A, *B, *D;
  cudaMalloc(&A, sizeof hA); cudaMalloc(&B, sizeof hB); cudaMalloc(&D, sizeof hD);
  cudaMemcpy(A, hA, sizeof hA, cudaMemcpyHostToDevice);
  cudaMemcpy(B, hB, sizeof hB, cudaMemcpyHostToDevice);
  k<<<1, 32>>>(A, B, D);
  cudaMemcpy(hD, D, sizeof hD, cudaMemcpyDeviceToHost);
  double err = 0;
  for (int i = 0; i < 128; ++i) err = std::fmax(err, std::fabs(hD[i] - ref[i]));
  printf("m16n8k4 f64 layout max err = %g (%s)\n", err, err < 1e-13 ? "LAYOUT OK" : "LAYOUT WRONG");
  return 0;
}
