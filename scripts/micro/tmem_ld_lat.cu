// TMEM load time per shape: 8 warps (two per SM sub-partition), each loading 8 KB (64 fp32
// per thread) and consuming every register, as the K3 softmax does for its S tile.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2505_07829_b200/csrc \
//        scripts/micro/tmem_ld_lat.cu -o scripts/micro/tmem_ld_lat
#include <cstdio>
#include <cstdint>
#include "sm100.cuh"
using namespace bfgpu::dev;

template <int SHAPE>
__global__ void bench(unsigned long long* out, float* sink) {
  __shared__ uint32_t slot;
  const uint32_t warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = slot;
  const uint32_t q = warp & 3, c = warp >> 2;
  float acc = 0.f;
  unsigned long long best = ~0ull;
  for (int it = 0; it < 64; ++it) {
    uint32_t r[64];
    __syncthreads();
    const unsigned long long t0 = clock64();
    if (SHAPE == 0) {  // 32x32b: this warp's 32 lanes, 32 columns of its half (8 KB as 2 x32 over 64 cols / 2 warps)
      const uint32_t ta = tmem + ((q * 32) << 16) + c * 64;
      tmem_ld_32x32b_x32(ta, *reinterpret_cast<uint32_t(*)[32]>(&r[0]));
      tmem_ld_32x32b_x32(ta + 32, *reinterpret_cast<uint32_t(*)[32]>(&r[32]));
    } else if (SHAPE == 1) {  // 16x256b: 16 lanes, 128 columns
      const uint32_t ta = tmem + ((q * 32 + c * 16) << 16);
      tmem_ld_16x256b_x8(ta, *reinterpret_cast<uint32_t(*)[32]>(&r[0]));
      tmem_ld_16x256b_x8(ta + 64, *reinterpret_cast<uint32_t(*)[32]>(&r[32]));
    } else {  // 16x32bx2: 16 lanes, two 64-column halves
      const uint32_t ta = tmem + ((q * 32 + c * 16) << 16);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        uint32_t* o = &r[32 * h];
        asm volatile(
            "tcgen05.ld.sync.aligned.16x32bx2.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
            "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32], 64;"
            : "=r"(o[0]), "=r"(o[1]), "=r"(o[2]), "=r"(o[3]), "=r"(o[4]), "=r"(o[5]), "=r"(o[6]), "=r"(o[7]), "=r"(o[8]),
              "=r"(o[9]), "=r"(o[10]), "=r"(o[11]), "=r"(o[12]), "=r"(o[13]), "=r"(o[14]), "=r"(o[15]), "=r"(o[16]),
              "=r"(o[17]), "=r"(o[18]), "=r"(o[19]), "=r"(o[20]), "=r"(o[21]), "=r"(o[22]), "=r"(o[23]), "=r"(o[24]),
              "=r"(o[25]), "=r"(o[26]), "=r"(o[27]), "=r"(o[28]), "=r"(o[29]), "=r"(o[30]), "=r"(o[31])
            : "r"(ta + 32 * h));
      }
    }
    tmem_wait_ld();
    float m = -1e30f;
#pragma unroll
    for (int k = 0; k < 64; ++k) m = fmaxf(m, __uint_as_float(r[k]));
    acc += m;
    const unsigned long long t1 = clock64();
    if (t1 - t0 < best) best = t1 - t0;
  }
  if (lane == 0) out[warp] = best;
  sink[threadIdx.x] = acc;
  tc_fence_before(); __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc<512>(tmem); }
}

int main() {
  unsigned long long* d; float* s; cudaMalloc(&d, 64); cudaMalloc(&s, 4096);
  const char* names[3] = {"32x32b (2 x32)", "16x256b (2 x8)", "16x32bx2 (2 x32)"};
  auto run = [&](auto kern, int k) {
    kern<<<1, 256>>>(d, s);
    unsigned long long h[8]; cudaMemcpy(h, d, 64, cudaMemcpyDeviceToHost);
    printf("%-18s err=%s  cycles per warp:", names[k], cudaGetErrorString(cudaGetLastError()));
    for (int w = 0; w < 8; ++w) printf(" %llu", h[w]);
    printf("\n");
  };
  run(bench<0>, 0); run(bench<1>, 1); run(bench<2>, 2);
}
