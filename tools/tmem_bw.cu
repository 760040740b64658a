// TMEM -> register read bandwidth per SM for the tcgen05.ld shapes an epilogue can use.
// One CTA per SM allocates 512 TMEM columns; W warps (W/4 per TMEM lane quarter) read it
// back ITERS times with one shape, each warp a different column range, and report the
// bytes read per SM clock (clock64 of the slowest warp).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_bw tools/tmem_bw.cu && ./tmem_bw
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

#define R32 "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}"
#define O32(r) "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), \
  "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),        \
  "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),      \
  "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])

// every shape moves 4 KB per warp instruction (32 registers per thread)
template <int SHAPE>
__device__ __forceinline__ void ld4k(uint32_t taddr, uint32_t (&r)[32]) {
  if constexpr (SHAPE == 0)
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 " R32 ", [%32];" : O32(r) : "r"(taddr));
  else if constexpr (SHAPE == 1)
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x8.b32 " R32 ", [%32];" : O32(r) : "r"(taddr));
  else if constexpr (SHAPE == 2)
    asm volatile("tcgen05.ld.sync.aligned.16x128b.x16.b32 " R32 ", [%32];" : O32(r) : "r"(taddr));
  else
    asm volatile("tcgen05.ld.sync.aligned.16x64b.x32.b32 " R32 ", [%32];" : O32(r) : "r"(taddr));
}

template <int SHAPE, int INFLIGHT>
__global__ void tmem_bw_kernel(int iters, unsigned long long* cycles, uint32_t* sink) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  const int nwarps = blockDim.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t base = slot;
  const int q = warp & 3;                 // the TMEM lane quarter this warp may access
  const int grp = warp >> 2;              // column group of this warp within its quarter
  const int ngrp = nwarps / 4;
  // 32x32b.x32 reads 32 columns; 16xNb shapes read 16 lanes (two halves of the quarter
  // alternate) x (4 KB / 16 lanes / 4 B) = 64 columns
  const int cols = SHAPE == 0 ? 32 : 64;
  const int span = 512 / ngrp;
  uint32_t acc = 0;
  __syncthreads();
  const long long t0 = clock64();
  for (int i = 0; i < iters; i += INFLIGHT) {
    uint32_t r[INFLIGHT][32];
#pragma unroll
    for (int j = 0; j < INFLIGHT; ++j) {
      const int it = i + j;
      const int col = grp * span + (it * cols) % span;
      const int lane_off = SHAPE == 0 ? 0 : ((it & 1) * 16);
      ld4k<SHAPE>(base + (static_cast<uint32_t>(q * 32 + lane_off) << 16) + col, r[j]);
    }
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int j = 0; j < INFLIGHT; ++j)
#pragma unroll
      for (int k = 0; k < 32; ++k) acc ^= r[j][k];
  }
  const long long t1 = clock64();
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if ((threadIdx.x & 31) == 0) atomicMax(&cycles[blockIdx.x], static_cast<unsigned long long>(t1 - t0));
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(base) : "memory");
}

template <int SHAPE, int INFLIGHT>
void run(const char* name, int warps, int sms) {
  const int iters = 4096;
  unsigned long long* d_cycles;
  uint32_t* d_sink;
  cudaMalloc(&d_cycles, sms * sizeof(unsigned long long));
  cudaMalloc(&d_sink, sms * warps * 32 * sizeof(uint32_t));
  cudaMemset(d_cycles, 0, sms * sizeof(unsigned long long));
  tmem_bw_kernel<SHAPE, INFLIGHT><<<sms, warps * 32>>>(iters, d_cycles, d_sink);  // warm-up
  cudaMemset(d_cycles, 0, sms * sizeof(unsigned long long));
  tmem_bw_kernel<SHAPE, INFLIGHT><<<sms, warps * 32>>>(iters, d_cycles, d_sink);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[256] = {0};
  cudaMemcpy(h, d_cycles, sms * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  unsigned long long mx = 0;
  for (int i = 0; i < sms; ++i) mx = h[i] > mx ? h[i] : mx;
  const double bytes = static_cast<double>(warps) * iters * 4096.0;
  printf("{\"shape\": \"%s\", \"warps\": %d, \"inflight\": %d, \"cycles\": %llu, \"bytes_per_clk_per_sm\": %.1f, \"err\": \"%s\"}\n",
         name, warps, INFLIGHT, mx, bytes / mx, cudaGetErrorString(e));
  cudaFree(d_cycles);
  cudaFree(d_sink);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int w : {4, 8, 16}) {
    run<0, 1>("32x32b.x32", w, sms);
    run<0, 2>("32x32b.x32", w, sms);
    run<1, 1>("16x256b.x8", w, sms);
    run<1, 2>("16x256b.x8", w, sms);
    run<2, 1>("16x128b.x16", w, sms);
    run<3, 1>("16x64b.x32", w, sms);
  }
  return 0;
}
