// Debug aid: times the L^{-1} kernels of librpchol_b200.so on a random well-conditioned L.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>
#include <cuda_runtime.h>
namespace rpcb {
void launch_linv(const double* lacc_cm, int m, int nb, int64_t ldl, int koff, double* linv_rm, cudaStream_t st);
}
int main(int argc, char** argv) {
  int m = argc > 1 ? atoi(argv[1]) : 116;
  std::vector<double> L((size_t)m * m, 0.0);
  srand(1);
  for (int c = 0; c < m; ++c)
    for (int a = c; a < m; ++a) L[(size_t)c * m + a] = a == c ? 1.0 + rand() / (double)RAND_MAX : 0.1 * (rand() / (double)RAND_MAX - 0.5);
  double *dL, *dI;
  cudaMalloc(&dL, sizeof(double) * m * m);
  cudaMalloc(&dI, sizeof(double) * 256 * 272);
  cudaMemcpy(dL, L.data(), sizeof(double) * m * m, cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int it = 0; it < 3; ++it) rpcb::launch_linv(dL, m, 256, 272, 0, dI, 0);
  cudaEventRecord(e0);
  for (int it = 0; it < 20; ++it) rpcb::launch_linv(dL, m, 256, 272, 0, dI, 0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("m=%d linv %.2f us per launch (%s)\n", m, ms * 1000 / 20, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
