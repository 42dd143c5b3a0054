// Fragment layouts of the 16-lane tcgen05.ld shapes, measured: TMEM lane l, column c is
// filled with (l << 8) | c through 32x32b stores, then read back through 16x64b / 16x128b /
// 16x256b loads; each thread prints which (lane, column) it received.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I paper_2505_07829_b200/csrc \
//        scripts/micro/tmem_layout.cu -o scripts/micro/tmem_layout
#include <cstdio>
#include <cstdint>
#include "sm100.cuh"
using namespace bfgpu::dev;

__global__ void layout(uint32_t* out) {
  __shared__ uint32_t slot;
  const uint32_t warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp == 0) tmem_alloc<32>(&slot);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = slot;
  const uint32_t lb = (warp * 32) << 16;
  uint32_t v[16];
  for (int c = 0; c < 16; ++c) v[c] = ((warp * 32 + lane) << 8) | c;
  tmem_st_32x32b_x16(tmem + lb, v);
  tmem_wait_st();
  __syncwarp();
  if (warp == 0) {
    uint32_t a, b0, b1, d0, d1, d2, d3, e0, e1, f0, f1;
    asm volatile("tcgen05.ld.sync.aligned.16x64b.x1.b32 {%0}, [%1];" : "=r"(a) : "r"(tmem));
    asm volatile("tcgen05.ld.sync.aligned.16x128b.x1.b32 {%0, %1}, [%2];" : "=r"(b0), "=r"(b1) : "r"(tmem));
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x1.b32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(d0), "=r"(d1), "=r"(d2), "=r"(d3) : "r"(tmem));
    asm volatile("tcgen05.ld.sync.aligned.16x64b.x2.b32 {%0, %1}, [%2];" : "=r"(e0), "=r"(e1) : "r"(tmem + (16u << 16)));
    asm volatile("tcgen05.ld.sync.aligned.16x32bx2.x2.b32 {%0, %1}, [%2], 4;" : "=r"(f0), "=r"(f1) : "r"(tmem));
    tmem_wait_ld();
    uint32_t* o = out + lane * 16;
    o[9] = f0; o[10] = f1;
    o[0] = a; o[1] = b0; o[2] = b1; o[3] = d0; o[4] = d1; o[5] = d2; o[6] = d3; o[7] = e0; o[8] = e1;
  }
  tc_fence_before(); __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc<32>(tmem); }
}

int main() {
  uint32_t* d; cudaMalloc(&d, 32 * 16 * 4); cudaMemset(d, 0xff, 32 * 16 * 4);
  layout<<<1, 128>>>(d);
  uint32_t h[32 * 16]; cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  const char* names[11] = {"16x64b.x1", "16x128b[0]", "16x128b[1]", "16x256b[0]", "16x256b[1]", "16x256b[2]", "16x256b[3]", "16x64b.x2@16[0]", "16x64b.x2@16[1]", "16x32bx2.x2,4[0]", "16x32bx2.x2,4[1]"};
  for (int k = 0; k < 11; ++k) {
    printf("%-16s", names[k]);
    for (int t = 0; t < 32; ++t) printf(" %u:%u", h[t * 16 + k] >> 8, h[t * 16 + k] & 255);
    printf("\n");
  }
}
