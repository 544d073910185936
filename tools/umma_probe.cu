// tools/umma_probe.cu — standalone check of k_pack_linv + k_var_umma
// (gadi_gpr_umma.cuh) against a binary64 host evaluation.
//   nvcc -O2 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/umma_probe tools/umma_probe.cu
//   tools/umma_probe [mp] [q]
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "../paper_2501_04229_b200/csrc/gadi_gpr_umma.cuh"
using namespace gpr_dev;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

int main(int argc, char** argv) {
  const int mp = argc > 1 ? atoi(argv[1]) : 512, q = argc > 2 ? atoi(argv[2]) : 512;
  const int m = mp - 37;  // exercise the k >= m mask
  const double ell = 1.0, sf2 = 3.8e-5, sn2 = 1e-4;
  std::mt19937_64 rng(5);
  std::uniform_real_distribution<double> U(0.0, 1.0);
  std::vector<double> X((size_t)mp * mp, 0.0), xs(mp), xq(q);
  for (int i = 0; i < mp; ++i) xs[i] = 9.2 + 9.2 * U(rng);
  for (int i = 0; i < q; ++i) xq[i] = 9.2 + 9.2 * U(rng);
  for (int i = 0; i < mp; ++i)
    for (int k = 0; k <= i; ++k) X[(size_t)i * mp + k] = (i == k ? 1.0 : -0.02 * U(rng)) * (i < m && k < m ? 1.0 : (i == k ? 1.0 : 0.0));
  std::vector<float2> xsf(mp), xqf(q);
  for (int i = 0; i < mp; ++i) { float h = (float)xs[i]; xsf[i] = make_float2(h, (float)(xs[i] - (double)h)); }
  for (int i = 0; i < q; ++i) { float h = (float)xq[i]; xqf[i] = make_float2(h, (float)(xq[i] - (double)h)); }
  double *dX, *dvar;
  float2 *dxs, *dxq;
  uint8_t* img;
  const int npass = mp / UM_PASS_ROWS;
  const size_t img_bytes = (size_t)4 * npass * (npass + 1) * UM_A_STAGE;
  CK(cudaMalloc(&dX, X.size() * 8));
  CK(cudaMalloc(&dvar, q * 8));
  CK(cudaMalloc(&dxs, mp * 8));
  CK(cudaMalloc(&dxq, q * 8));
  CK(cudaMalloc(&img, img_bytes));
  CK(cudaMemcpy(dX, X.data(), X.size() * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dxs, xsf.data(), mp * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dxq, xqf.data(), q * 8, cudaMemcpyHostToDevice));
  k_pack_linv<<<dim3(8 * npass, npass), 256>>>(dX, mp, mp, 64.0, img);
  CK(cudaGetLastError());
  CK(cudaFuncSetAttribute(k_var_umma, cudaFuncAttributeMaxDynamicSharedMemorySize, UM_SMEM));
  const double sfsn = 1e7 * sf2 + sn2;  // large: the probe's X is not an inverse factor, keep var > 0
  VarParams P{img, dxs, dxq, mp, m, q, (float)(1.0 / ell), sf2 / 268435456.0, sfsn, dvar};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    k_var_umma<<<(q + UM_NQ - 1) / UM_NQ, UM_THREADS, UM_SMEM>>>(P);
    cudaEventRecord(e1);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 3.0 * 2.0 * (double)mp * mp / 2 * q;
    printf("k_var_umma mp=%d q=%d: %.3f ms, %.1f TFLOP/s (3-term, triangular)\n", mp, q, ms, flops / ms / 1e9);
  }
  std::vector<double> var(q);
  CK(cudaMemcpy(var.data(), dvar, q * 8, cudaMemcpyDeviceToHost));
  double worst = 0, worst_s = 0;
  const int ncheck = q < 64 ? q : 64;
  for (int t = 0; t < ncheck; ++t) {
    const int j = (int)((long long)t * q / ncheck);
    std::vector<double> k(mp, 0.0);
    for (int i = 0; i < m; ++i) { const double d = (xq[j] - xs[i]) / ell; k[i] = exp(-0.5 * d * d); }
    double s = 0;
    for (int i = 0; i < mp; ++i) {
      double acc = 0;
      for (int c = 0; c <= i; ++c) acc += X[(size_t)i * mp + c] * k[c];
      s += acc * acc;
    }
    const double want = sfsn - sf2 * s, got = var[j];
    const double gs = (sfsn - got) / sf2;
    worst = fmax(worst, fabs(got - want) / fabs(want));
    worst_s = fmax(worst_s, fabs(gs - s) / s);
    if (t < 4) printf("  q %d: sum want %.9e got %.9e  var want %.9e got %.9e\n", j, s, gs, want, got);
  }
  printf("max rel err: var %.3e, sum of squares %.3e  %s\n", worst, worst_s, worst_s < 1e-4 ? "OK" : "FAIL");
  return worst_s < 1e-4 ? 0 : 2;
}
