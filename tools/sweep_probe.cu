// Debug aid: times the rejection sweep (sweep.cu, compiled in with RPC_SWEEP_PROBE) on a
// Gaussian-kernel H of b random points, with per-16-block phase clocks:
// decisions (warp 0), panel + L-column writes, trailing update.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DRPC_SWEEP_PROBE
//        -I paper_2410_03969_b200/csrc -o tools/sweep_probe tools/sweep_probe.cu
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "sweep.cu"

int main(int argc, char** argv) {
  const int b = argc > 1 ? atoi(argv[1]) : 120;
  const int d = argc > 2 ? atoi(argv[2]) : 30;
  const double sigma = argc > 3 ? atof(argv[3]) : 3.0;
  const double spread = argc > 4 ? atof(argv[4]) : 3.0;
  std::vector<double> x((size_t)b * d), H((size_t)b * b), prop((size_t)b * 2);
  srand(7);
  for (auto& v : x) v = (rand() / (double)RAND_MAX - 0.5) * spread;
  for (int p = 0; p < b; ++p) {
    prop[2 * p] = p;
    for (int q = 0; q < b; ++q) {
      double dd = 0;
      for (int j = 0; j < d; ++j) dd += (x[p * d + j] - x[q * d + j]) * (x[p * d + j] - x[q * d + j]);
      H[(size_t)p * b + q] = exp(-0.5 * dd / (sigma * sigma));
    }
  }
  double *dH, *dprop, *lcol, *lacc, *hp;
  int* pos;
  int64_t* ids;
  rpcb::SweepOut* out;
  cudaMalloc(&dH, sizeof(double) * b * b);
  cudaMalloc(&dprop, sizeof(double) * b * 2);
  cudaMalloc(&lcol, sizeof(double) * b * b);
  cudaMalloc(&lacc, sizeof(double) * b * b);
  cudaMalloc(&hp, sizeof(double) * b * b);
  cudaMalloc(&pos, sizeof(int) * b);
  cudaMalloc(&ids, sizeof(int64_t) * b);
  cudaMalloc(&out, sizeof(rpcb::SweepOut));
  cudaMemcpy(dH, H.data(), sizeof(double) * b * b, cudaMemcpyHostToDevice);
  cudaMemcpy(dprop, prop.data(), sizeof(double) * b * 2, cudaMemcpyHostToDevice);
  rpcb::RecordLayout lay{2, 2, 2};
  auto run = [&] { rpcb::launch_sweep(dH, b, 0, 0, dprop, lay, pos, ids, lcol, lacc, out, hp, 0); };
  for (int i = 0; i < 3; ++i) run();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int i = 0; i < 20; ++i) run();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  rpcb::SweepOut o;
  cudaMemcpy(&o, out, sizeof(o), cudaMemcpyDeviceToHost);
  unsigned long long clk[32][4];
  cudaMemcpyFromSymbol(clk, rpcb::g_sweep_clk, sizeof(clk));
  printf("b=%d accepted m=%d: %.2f us per sweep (%s)\n", b, o.m, ms * 1000 / 20,
         cudaGetErrorString(cudaGetLastError()));
  double dec = 0, pan = 0, trl = 0;
  const int nblk = (b + 15) / 16;
  for (int k = 0; k < nblk; ++k) {
    dec += clk[k][1] - clk[k][0];
    pan += clk[k][2] - clk[k][1];
    trl += clk[k][3] - clk[k][2];
  }
  printf("cycles: decisions %.0f  panel+lcol %.0f  trailing %.0f  (sum %.0f; first block start -> last end %llu)\n",
         dec, pan, trl, dec + pan + trl, clk[nblk - 1][3] - clk[0][0]);
  unsigned long long st[256][4];
  cudaMemcpyFromSymbol(st, rpcb::g_step_clk, sizeof(st));
  for (int i = 0; i < b && i < 40; ++i)
    printf("step %3d: sqrt+div %6lld  hnext %6lld  rest %6lld  start->next start %6lld\n", i,
           (long long)(st[i][2] - st[i][0]), (long long)(st[i][3] - st[i][2]), (long long)(st[i][1] - st[i][3]),
           i + 1 < b ? (long long)(st[i + 1][0] - st[i][0]) : 0LL);
  return 0;
}
