// write_pat.cu -- which write pattern lets s2_out (b rows of many instances) approach the HBM
// write ceiling?  1000 rows x ~5 MB (one config-5 trace: 2.5e6 u16 requests per instance row),
// CTAs of 256 threads each own a group of G rows and an event range; variants:
//   il  : s2_out's pattern -- per 8-event tile (4 KB per row), cycle over the G rows
//   seq : per row, write the CTA's whole range (R events) before the next row (1 open row per CTA)
//   tma : seq, but each row chunk is staged in shared memory and written by cp.async.bulk
// grid order: groups fastest (gx = groups) or ranges fastest.
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o /tmp/write_pat tools/write_pat.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__global__ void __launch_bounds__(256) il_kernel(uint16_t* out, size_t row_len, uint32_t G, uint32_t R,
                                                 bool groups_fast, uint32_t ngroups) {
  const uint32_t grp = groups_fast ? blockIdx.x : blockIdx.y, rng = groups_fast ? blockIdx.y : blockIdx.x;
  const size_t e0 = size_t(rng) * R, e1 = min(row_len, e0 + R);
  const uint4 v = make_uint4(threadIdx.x, 1, 2, 3);
  for (size_t e = e0 + 8 * threadIdx.x; e < e1; e += 8 * 256)
    for (uint32_t i = 0; i < G; ++i) *reinterpret_cast<uint4*>(out + (size_t(grp) * G + i) * row_len + e) = v;
}

__global__ void __launch_bounds__(256) seq_kernel(uint16_t* out, size_t row_len, uint32_t G, uint32_t R,
                                                  bool groups_fast, uint32_t ngroups) {
  const uint32_t grp = groups_fast ? blockIdx.x : blockIdx.y, rng = groups_fast ? blockIdx.y : blockIdx.x;
  const size_t e0 = size_t(rng) * R, e1 = min(row_len, e0 + R);
  const uint4 v = make_uint4(threadIdx.x, 1, 2, 3);
  for (uint32_t i = 0; i < G; ++i)
    for (size_t e = e0 + 8 * threadIdx.x; e < e1; e += 8 * 256)
      *reinterpret_cast<uint4*>(out + (size_t(grp) * G + i) * row_len + e) = v;
}

// staged rows: the CTA computes a row chunk of R events into smem (here: a constant), then one
// thread issues a bulk store of it; double buffered over 2 x R x 2 bytes of shared memory
__global__ void __launch_bounds__(256) tma_kernel(uint16_t* out, size_t row_len, uint32_t G, uint32_t R,
                                                  bool groups_fast, uint32_t ngroups) {
  extern __shared__ __align__(128) uint4 stile[];
  const uint32_t grp = groups_fast ? blockIdx.x : blockIdx.y, rng = groups_fast ? blockIdx.y : blockIdx.x;
  const size_t e0 = size_t(rng) * R, e1 = min(row_len, e0 + R);
  const uint32_t n16 = static_cast<uint32_t>((e1 - e0) / 8);
  for (uint32_t i = 0; i < G; ++i) {
    uint4* buf = stile + (i & 1) * (R / 8);
    if (threadIdx.x == 0 && i >= 2) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    __syncthreads();
    for (uint32_t k = threadIdx.x; k < n16; k += 256) buf[k] = make_uint4(k, i, 2, 3);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
      const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(buf));
      uint16_t* dst = out + (size_t(grp) * G + i) * row_len + e0;
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(s), "r"(n16 * 16)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
  const size_t row_len = 2500000 / 8 * 8;  // u16 per row (16-byte aligned rows)
  const uint32_t rows = 992;
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
    printf("%-44s %.3f ms  %6.0f GB/s %s\n", name, best, bytes / best / 1e6, e ? cudaGetErrorString(e) : "");
  };
  for (uint32_t G : {1u, 4u, 8u, 16u, 32u}) {
    const uint32_t ng = rows / G;
    for (uint32_t R : {4096u, 16384u, 32768u}) {
      const uint32_t nr = static_cast<uint32_t>((row_len + R - 1) / R);
      for (int gf = 1; gf >= 0; --gf) {
        dim3 grid = gf ? dim3(ng, nr) : dim3(nr, ng);
        char nm[96];
        snprintf(nm, sizeof nm, "il  G=%2u R=%5u %s", G, R, gf ? "groups-fast" : "ranges-fast");
        run(nm, [&] { il_kernel<<<grid, 256>>>(buf, row_len, G, R, gf, ng); });
        snprintf(nm, sizeof nm, "seq G=%2u R=%5u %s", G, R, gf ? "groups-fast" : "ranges-fast");
        run(nm, [&] { seq_kernel<<<grid, 256>>>(buf, row_len, G, R, gf, ng); });
        if (R <= 16384) {
          const int sm = 2 * R * 2;
          cudaFuncSetAttribute(tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
          snprintf(nm, sizeof nm, "tma G=%2u R=%5u %s", G, R, gf ? "groups-fast" : "ranges-fast");
          run(nm, [&] { tma_kernel<<<grid, 256, sm>>>(buf, row_len, G, R, gf, ng); });
        }
      }
    }
  }
  cudaMemsetAsync(buf, 0, row_len * rows * 2);
  run("cudaMemsetAsync", [&] { cudaMemsetAsync(buf, 0, row_len * rows * 2); });
  return 0;
}
