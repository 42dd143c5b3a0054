// Pipeline study for K3: builds attention.cu with BF_ATTN_TRACE and prints per-block
// SM-clock phase stamps of CTA 0 (softmax WG0/WG1 and the MMA issuer).
//   cd paper_2505_07829_b200/csrc && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DBF_ATTN_TRACE
//        -I ../../include -I . ../../scripts/micro/attn_trace.cu $(ls *.cu | grep -v '^attention.cu$')
//        -o ../../scripts/micro/attn_trace -lcuda -ldl -lpthread
#include <cstdio>
#include <vector>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include "../../paper_2505_07829_b200/csrc/attention.cu"


int main() {
  const int BH = 256, S = 2048, D = 128;
  size_t n = size_t(BH) * S * D;
  void *Q, *K, *V, *O;
  cudaMalloc(&Q, n * 2); cudaMalloc(&K, n * 2); cudaMalloc(&V, n * 2); cudaMalloc(&O, n * 2);
  std::vector<uint16_t> h(n);
  uint32_t st = 12345;
  const bool gauss = getenv("TRACE_GAUSS") != nullptr;  // N(0,1) like torch.randn, else U(-1.7, 1.7)
  for (auto& x : h) {
    st = st * 1664525u + 1013904223u;
    float u1 = ((st >> 9) + 0.5f) * (1.0f / 8388608.0f);
    st = st * 1664525u + 1013904223u;
    float u2 = (st >> 9) * (1.0f / 8388608.0f);
    float f = gauss ? sqrtf(-2.f * logf(u1)) * cosf(6.2831853f * u2) : (u1 - 0.5f) * 3.4f;
    uint32_t b; memcpy(&b, &f, 4); x = uint16_t(b >> 16);
  }
  cudaMemcpy(Q, h.data(), n * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(K, h.data(), n * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(V, h.data(), n * 2, cudaMemcpyHostToDevice);
  unsigned long long* tr;
  cudaMalloc(&tr, 4 * 64 * 8 * 8);
  cudaMemset(tr, 0, 4 * 64 * 8 * 8);
  bfgpu::attn::attn_trace_buffer = tr;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int it = 0; it < 3; ++it) bfgpu::attention_bf16(Q, K, V, O, BH, S, S, D, D, 0.f, 0, nullptr, 0, 0);
  cudaEventRecord(e0);
  for (int it = 0; it < 5; ++it) bfgpu::attention_bf16(Q, K, V, O, BH, S, S, D, D, 0.f, 0, nullptr, 0, 0);
  cudaEventRecord(e1);
  cudaDeviceSynchronize();
  float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 5;
  printf("err=%s  %.3f ms  %.1f TFLOP/s\n", cudaGetErrorString(cudaGetLastError()), ms, 4.0 * BH * S * S * D / ms / 1e9);
  std::vector<unsigned long long> t(4 * 64 * 8);
  cudaMemcpy(t.data(), tr, t.size() * 8, cudaMemcpyDeviceToHost);
  unsigned long long base = t[(0 * 64 + 10) * 8 + 0];
  printf("softmax (warp 0) per sub-tile: wait S_ready max_done half0_arrived half1_arrived | MMA issuer i: p_seen token pv_issued qk_issued commits_done\n");
  for (int g = 10; g < 22; ++g) {
    auto v = [&](int slot, int k) { return (long long)(t[(slot * 64 + g) * 8 + k] - base); };
    printf("%3d | T0 %6lld %6lld %6lld %6lld %6lld | T1 %6lld %6lld %6lld %6lld %6lld | M0 %6lld %6lld %6lld %6lld %6lld | M1 %6lld %6lld %6lld %6lld %6lld\n",
           g, v(0, 0), v(0, 1), v(0, 2), v(0, 3), v(0, 4), v(1, 0), v(1, 1), v(1, 2), v(1, 3), v(1, 4), v(2, 0), v(2, 2),
           v(2, 3), v(2, 4), v(2, 1), v(3, 0), v(3, 2), v(3, 3), v(3, 4), v(3, 1));
  }
#ifdef BF_ATTN_TRACE_LD
  for (int g = 16; g < 22; ++g) {
    auto v = [&](int slot, int k) { return (long long)(t[(slot * 64 + g) * 8 + k] - base); };
    printf("%3d S_ready->loaded->max: T0 %lld %lld | T1 %lld %lld\n", g, v(0, 5) - v(0, 1), v(0, 2) - v(0, 5), v(1, 5) - v(1, 1), v(1, 2) - v(1, 5));
  }
#endif
  printf("epilogue warpgroup, second tile (T0 | T1): enter o_full_seen stored\n");
  {
    auto v = [&](int slot, int k) { return (long long)(t[(slot * 64 + 1) * 8 + k] - base); };
    printf("    %6lld %6lld %6lld | %6lld %6lld %6lld\n", v(0, 5), v(0, 6), v(0, 7), v(1, 5), v(1, 6), v(1, 7));
  }
}
