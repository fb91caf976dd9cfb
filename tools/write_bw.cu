// write_bw.cu -- write-only HBM bandwidth on this GPU, for the roofline of write-dominated
// kernels (s2_out writes ~2 bytes per simulated request and reads ~0.13).
// Variants: cudaMemsetAsync, STG.128 (default / .cs streaming / .wb), TMA bulk store
// (cp.async.bulk.global.shared::cta) from a shared-memory tile, and STG.128 into many
// interleaved rows (s2_out's pattern: each CTA writes 4 KB pieces of ~35 rows).
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o /tmp/write_bw tools/write_bw.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e = (x);                                                        \
    if (e != cudaSuccess) {                                                     \
      printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e));          \
      return 1;                                                                 \
    }                                                                           \
  } while (0)

template <int MODE>
__global__ void __launch_bounds__(256) stg_kernel(uint4* out, size_t n16) {
  const uint4 v = make_uint4(threadIdx.x, 1, 2, 3);
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n16; i += size_t(gridDim.x) * blockDim.x) {
    if (MODE == 0) out[i] = v;
    if (MODE == 1) __stcs(out + i, v);
    if (MODE == 2) __stwt(out + i, v);
  }
}

// rows: `rows` rows of `row16` uint4 each; CTA (r, y) writes rows [y*G, y*G+G) over event range r
__global__ void __launch_bounds__(256) rows_kernel(uint4* out, size_t row16, uint32_t G, uint32_t range16) {
  const uint4 v = make_uint4(threadIdx.x, 1, 2, 3);
  const size_t e0 = size_t(blockIdx.x) * range16;
  for (size_t e = e0 + threadIdx.x; e < e0 + range16 && e < row16; e += blockDim.x)
    for (uint32_t i = 0; i < G; ++i) out[(size_t(blockIdx.y) * G + i) * row16 + e] = v;
}

// rows2: like rows_kernel, but per 'visit' a CTA writes V consecutive 4 KB tiles to each of SB
// rows before the next SB rows (SB = G, V = 1 is rows_kernel).  gy_fast swaps the grid order.
__global__ void __launch_bounds__(256) rows2_kernel(uint4* out, size_t row16, uint32_t G, uint32_t range16,
                                                     uint32_t SB, uint32_t V, bool gy_fast) {
  const uint4 val = make_uint4(threadIdx.x, 1, 2, 3);
  const uint32_t r = gy_fast ? blockIdx.y : blockIdx.x, grp = gy_fast ? blockIdx.x : blockIdx.y;
  const size_t e0 = size_t(r) * range16, e1 = e0 + range16 < row16 ? e0 + range16 : row16;
  for (size_t base = e0; base < e1; base += size_t(V) * blockDim.x)
    for (uint32_t sb = 0; sb < G; sb += SB)
      for (uint32_t i = sb; i < sb + SB && i < G; ++i)
        for (uint32_t v = 0; v < V; ++v) {
          const size_t e = base + v * blockDim.x + threadIdx.x;
          if (e < e1) out[(size_t(grp) * G + i) * row16 + e] = val;
        }
}

// rows3: rows of `len16` uint4 at stride `stride16` (padding between rows), V = 4 tiles per visit
__global__ void __launch_bounds__(256) rows3_kernel(uint4* out, size_t len16, size_t stride16, uint32_t G,
                                                     uint32_t range16) {
  const uint4 val = make_uint4(threadIdx.x, 1, 2, 3);
  const size_t e0 = size_t(blockIdx.x) * range16, e1 = e0 + range16 < len16 ? e0 + range16 : len16;
  for (size_t base = e0; base < e1; base += 4 * blockDim.x)
    for (uint32_t i = 0; i < G; ++i)
      for (uint32_t v = 0; v < 4; ++v) {
        const size_t e = base + v * blockDim.x + threadIdx.x;
        if (e < e1) out[(size_t(blockIdx.y) * G + i) * stride16 + e] = val;
      }
}

// rows4: CTA (r, grp) of NR CTAs per group takes the interleaved tiles r, r + NR, ... (tile =
// T uint4 per row), all G rows per tile: the CTAs of a group move through the rows together
__global__ void __launch_bounds__(256) rows4_kernel(uint4* out, size_t len16, uint32_t G, uint32_t T) {
  const uint4 val = make_uint4(threadIdx.x, 1, 2, 3);
  const uint32_t NR = gridDim.x;
  for (size_t t0 = size_t(blockIdx.x) * T; t0 < len16; t0 += size_t(NR) * T)
    for (uint32_t i = 0; i < G; ++i)
      for (uint32_t v = threadIdx.x; v < T; v += blockDim.x) {
        const size_t e = t0 + v;
        if (e < len16) out[(size_t(blockIdx.y) * G + i) * len16 + e] = val;
      }
}

__global__ void __launch_bounds__(128) tma_kernel(char* out, size_t bytes, uint32_t chunk) {
  extern __shared__ __align__(128) char tile[];
  for (uint32_t k = threadIdx.x; k < chunk / 16; k += blockDim.x)
    reinterpret_cast<uint4*>(tile)[k] = make_uint4(k, 1, 2, 3);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(tile));
    for (size_t off = size_t(blockIdx.x) * chunk; off + chunk <= bytes; off += size_t(gridDim.x) * chunk) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(out + off), "r"(s), "r"(chunk)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 4;" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}

int main() {
  const size_t bytes = 5000000000ull;
  char* buf;
  CK(cudaMalloc(&buf, bytes));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto run = [&](const char* name, auto fn) {
    fn();
    cudaDeviceSynchronize();
    float best = 1e9f;
    for (int r = 0; r < 10; ++r) {
      cudaEventRecord(a);
      fn();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    cudaError_t e = cudaGetLastError();
    printf("%-34s %.3f ms  %6.0f GB/s%s\n", name, best, bytes / best / 1e6, e ? cudaGetErrorString(e) : "");
  };
  const size_t n16 = bytes / 16;
  run("cudaMemsetAsync", [&] { cudaMemsetAsync(buf, 0, bytes); });
  for (int g : {148 * 4, 148 * 8, 148 * 16, 148 * 64}) {
    char nm[64];
    snprintf(nm, sizeof nm, "STG.128 grid %d", g);
    run(nm, [&] { stg_kernel<0><<<g, 256>>>(reinterpret_cast<uint4*>(buf), n16); });
  }
  run("STG.128 .cs grid 1184", [&] { stg_kernel<1><<<1184, 256>>>(reinterpret_cast<uint4*>(buf), n16); });
  run("STG.128 .wt grid 1184", [&] { stg_kernel<2><<<1184, 256>>>(reinterpret_cast<uint4*>(buf), n16); });
  for (uint32_t G : {1u, 8u, 35u}) {
    const uint32_t rows = 1000 / G * G;
    const size_t row16 = n16 / rows;
    const uint32_t range16 = 31744 / 8;  // s2_out: 31744 events per CTA, 8 events per uint4
    const dim3 grid((row16 + range16 - 1) / range16, rows / G);
    char nm[64];
    snprintf(nm, sizeof nm, "rows G=%u grid %ux%u", G, grid.x, grid.y);
    run(nm, [&] { rows_kernel<<<grid, 256>>>(reinterpret_cast<uint4*>(buf), row16, G, range16); });
  }
  for (uint32_t G : {8u, 35u, 64u}) {
    const uint32_t rows = 950 / G * G;
    const size_t len16 = 4999184 / 16;  // one config-5 trace: ~2.5e6 u16 requests per row
    for (size_t pad : {0ul, 256ul, 2048ul, 4352ul, 66304ul, 1048576ul}) {
      const size_t stride16 = len16 + pad / 16;
      if (stride16 * 16 * rows > bytes) continue;
      const uint32_t R = 31744 / 8;
      const dim3 grid((len16 + R - 1) / R, rows / G);
      char nm[96];
      snprintf(nm, sizeof nm, "rows3 G=%u pad=%zu", G, pad);
      const double wb = double(len16) * 16 * rows;
      cudaEventRecord(a);
      rows3_kernel<<<grid, 256>>>(reinterpret_cast<uint4*>(buf), len16, stride16, G, R);
      cudaDeviceSynchronize();
      float best = 1e9f;
      for (int r = 0; r < 10; ++r) {
        cudaEventRecord(a);
        rows3_kernel<<<grid, 256>>>(reinterpret_cast<uint4*>(buf), len16, stride16, G, R);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
      }
      printf("%-34s %.3f ms  %6.0f GB/s\n", nm, best, wb / best / 1e6);
    }
  }
  for (uint32_t G : {8u, 35u, 64u}) {
    const uint32_t rows = 950 / G * G;
    const size_t len16 = 4999184 / 16;
    const double wb = double(len16) * 16 * rows;
    for (uint32_t NR : {40u, 79u, 160u})
      for (uint32_t T : {256u, 1024u}) {
        const dim3 grid(NR, rows / G);
        float best = 1e9f;
        for (int r = 0; r < 11; ++r) {
          cudaEventRecord(a);
          rows4_kernel<<<grid, 256>>>(reinterpret_cast<uint4*>(buf), len16, G, T);
          cudaEventRecord(b);
          cudaEventSynchronize(b);
          float ms;
          cudaEventElapsedTime(&ms, a, b);
          if (r && ms < best) best = ms;
        }
        printf("rows4 G=%u NR=%u T=%u KB  %.3f ms  %6.0f GB/s\n", G, NR, T * 16 / 1024, best, wb / best / 1e6);
      }
  }
  for (uint32_t chunk : {16384u, 32768u}) {
    cudaFuncSetAttribute(tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, chunk);
    char nm[64];
    snprintf(nm, sizeof nm, "TMA bulk store %u B x 592", chunk);
    run(nm, [&] { tma_kernel<<<592, 128, chunk>>>(buf, bytes, chunk); });
    snprintf(nm, sizeof nm, "TMA bulk store %u B x 1184", chunk);
    run(nm, [&] { tma_kernel<<<1184, 128, chunk>>>(buf, bytes, chunk); });
  }
  return 0;
}
