// Write-pattern microbenchmark for s2_out's writer groups (992 rows x 2.5e6 u16, G = 16 rows per CTA):
//   cur : s2_out's pattern -- CTA = (group, range of R events); per tile of 2048 events the rows go
//         WB at a time through a WS-slot stage (2 CTA barriers per batch), 4 KB bulk store per row
//   row : row-major -- CTA = (group, range of R events); per row the whole range is staged (R x 2 B)
//         in a ring of S slots and written by ONE bulk store (R x 2 B contiguous per row)
// Extra dynamic smem `pad` emulates the per-event inputs staged beside the ring.
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o /tmp/writer_pat tools/writer_pat.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ void bulk_store(void* dst, const void* src, uint32_t bytes) {
  const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(src));
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(sa), "r"(bytes) : "memory");
}

template <int WB, int WS>
__global__ void __launch_bounds__(256) cur_kernel(uint16_t* out, size_t row_len, uint32_t G, uint32_t R) {
  extern __shared__ __align__(128) uint4 stg[];
  const uint32_t grp = blockIdx.x, rng = blockIdx.y, t = threadIdx.x;
  const size_t e0 = size_t(rng) * R, e1 = min(row_len, e0 + R);
  uint32_t it = 0;
  for (size_t base = e0; base < e1; base += 2048) {
    const uint32_t nv = static_cast<uint32_t>((min(e1, base + 2048) - base) / 8);
    for (uint32_t rb = 0; rb < G; rb += WB, ++it) {
      const uint32_t sl = it % WS;
      if (it >= WS && t < G) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(WS - 1) : "memory");
      __syncthreads();
      for (uint32_t q = 0; q < WB && rb + q < G; ++q) stg[(sl * WB + q) * 256 + t] = make_uint4(t, q, rb, it);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
      if (t >= rb && t < rb + WB && t < G)
        bulk_store(out + (size_t(grp) * G + t) * row_len + base, stg + (sl * WB + (t - rb)) * 256, nv * 16);
      if (t < G) asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  if (t < G) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <int S>
__global__ void __launch_bounds__(256) row_kernel(uint16_t* out, size_t row_len, uint32_t G, uint32_t R) {
  extern __shared__ __align__(128) uint4 ring[];
  const uint32_t grp = blockIdx.x, rng = blockIdx.y, t = threadIdx.x;
  const size_t e0 = size_t(rng) * R, e1 = min(row_len, e0 + R);
  const uint32_t nv = static_cast<uint32_t>((e1 - e0) / 8), sv = R / 8;
  for (uint32_t i = 0; i < G; ++i) {
    uint4* slot = ring + (i % S) * sv;
    if (i >= S && t == 0) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(S - 1) : "memory");
    __syncthreads();
    for (uint32_t v = t; v < nv; v += 256) slot[v] = make_uint4(v, i, 2, 3);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (t == 0) {
      bulk_store(out + (size_t(grp) * G + i) * row_len + e0, slot, nv * 16);
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  if (t == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
  const size_t row_len = 2500000 / 8 * 8;
  const uint32_t rows = 992, G = 16, ng = rows / G;
  uint16_t* buf;
  if (cudaMalloc(&buf, row_len * rows * 2) != cudaSuccess) return 1;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const double bytes = double(row_len) * rows * 2;
  auto run = [&](const char* name, auto launch) {
    launch();
    cudaDeviceSynchronize();
    float best = 1e9f;
    for (int r = 0; r < 8; ++r) {
      cudaEventRecord(a);
      launch();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      best = ms < best ? ms : best;
    }
    cudaError_t e = cudaGetLastError();
    printf("%-48s %.3f ms  %6.0f GB/s %s\n", name, best, bytes / best / 1e6, e ? cudaGetErrorString(e) : "");
  };
  char nm[128];
  auto cur = [&](auto kern, int WB, int WS, uint32_t R) {
    const uint32_t nr = static_cast<uint32_t>((row_len + R - 1) / R);
    const int sm = WS * WB * 4096;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    snprintf(nm, sizeof nm, "cur WB=%d WS=%d R=%u", WB, WS, R);
    run(nm, [&] { kern<<<dim3(ng, nr), 256, sm>>>(buf, row_len, G, R); });
  };
  for (uint32_t R : {31744u, 8192u, 4096u}) {
    cur(cur_kernel<6, 2>, 6, 2, R);
    cur(cur_kernel<1, 4>, 1, 4, R);
    cur(cur_kernel<1, 8>, 1, 8, R);
    cur(cur_kernel<2, 4>, 2, 4, R);
    cur(cur_kernel<4, 3>, 4, 3, R);
    cur(cur_kernel<16, 1>, 16, 1, R);
  }
  for (uint32_t R : {4096u}) {
    const uint32_t nr = static_cast<uint32_t>((row_len + R - 1) / R);
    for (uint32_t pad : {0u, 24576u}) {
      {
        const int sm = 2 * R * 2 + pad;
        cudaFuncSetAttribute(row_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
        snprintf(nm, sizeof nm, "row S=2 R=%u pad=%u", R, pad);
        run(nm, [&] { row_kernel<2><<<dim3(ng, nr), 256, sm>>>(buf, row_len, G, R); });
      }
      {
        const int sm = 3 * R * 2 + pad;
        cudaFuncSetAttribute(row_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
        snprintf(nm, sizeof nm, "row S=3 R=%u pad=%u", R, pad);
        run(nm, [&] { row_kernel<3><<<dim3(ng, nr), 256, sm>>>(buf, row_len, G, R); });
      }
    }
  }
  return 0;
}
