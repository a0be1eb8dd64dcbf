// stream_probe.cu — calibration of the decode kernels' data movement: how fast can N CTAs (one
// per SM) stream HBM -> shared memory with a single producer thread issuing cp.async.bulk into a
// ring of S slots of B bytes, when the consumer frees each slot as soon as it lands?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/stream_probe tools/stream_probe.cu
//   /tmp/stream_probe
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void minit(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mexpect(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void marrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mwait(uint64_t* b, uint32_t ph) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile("{\n .reg .pred P;\n mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n selp.u32 %0, 1, 0, P;\n}\n"
                 : "=r"(ok)
                 : "r"(su32(b)), "r"(ph)
                 : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t n, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(dst)),
               "l"(src), "r"(n), "r"(su32(bar))
               : "memory");
}

// per CTA: `bytes` contiguous bytes starting at src + blockIdx.x * bytes, ring of S slots of B
// bytes; chunk = the bulk-copy size (a slot is filled by B / chunk copies)
__global__ void __launch_bounds__(64, 1) probe(const uint8_t* src, int64_t bytes, int S, int B, int chunk, int* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + static_cast<size_t>(S) * B);
  uint64_t* empty = full + S;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      minit(&full[s], 1);
      minit(&empty[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint8_t* base = src + blockIdx.x * bytes;
  const int n = static_cast<int>(bytes / B);
  if (threadIdx.x == 32) {  // producer
    for (int k = 0; k < n; ++k) {
      const int s = k % S;
      if (k >= S) mwait(&empty[s], ((k / S) & 1) ^ 1);
      mexpect(&full[s], B);
      for (int c = 0; c < B; c += chunk) bulk(sm + static_cast<size_t>(s) * B + c, base + static_cast<int64_t>(k) * B + c, chunk, &full[s]);
    }
  } else if (threadIdx.x == 0) {  // consumer: touch one word, free the slot
    int acc = 0;
    for (int k = 0; k < n; ++k) {
      const int s = k % S;
      mwait(&full[s], (k / S) & 1);
      acc += sm[static_cast<size_t>(s) * B];
      marrive(&empty[s]);
    }
    if (acc == 12345) *sink = acc;
  }
}

// B: P producer lanes of one warp; lane p owns the sub-ring of slots [p*S/P, (p+1)*S/P) and the
// sequence numbers k = p (mod P); one consumer lane per sub-ring frees each slot as it lands
__global__ void __launch_bounds__(64, 1) probe_lanes(const uint8_t* src, int64_t bytes, int S, int B, int P, int* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + static_cast<size_t>(S) * B);
  uint64_t* empty = full + S;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      minit(&full[s], 1);
      minit(&empty[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint8_t* base = src + blockIdx.x * bytes;
  const int n = static_cast<int>(bytes / B);
  const int spp = S / P;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x >= 32 && lane < P) {  // producers
    int j = 0;
    for (int k = lane; k < n; k += P, ++j) {
      const int s = lane * spp + j % spp;
      if (j >= spp) mwait(&empty[s], ((j / spp) & 1) ^ 1);
      mexpect(&full[s], B);
      bulk(sm + static_cast<size_t>(s) * B, base + static_cast<int64_t>(k) * B, B, &full[s]);
    }
  } else if (threadIdx.x < 32 && lane < P) {  // consumers
    int acc = 0, j = 0;
    for (int k = lane; k < n; k += P, ++j) {
      const int s = lane * spp + j % spp;
      mwait(&full[s], (j / spp) & 1);
      acc += sm[static_cast<size_t>(s) * B];
      marrive(&empty[s]);
    }
    if (acc == 12345) *sink = acc;
  }
}

// C: plain 16-byte loads by W warps, U loads in flight per lane (registers), summed
template <int U>
__global__ void __launch_bounds__(256, 1) probe_ldg(const uint8_t* src, int64_t bytes, int* sink) {
  const uint4* base = reinterpret_cast<const uint4*>(src + blockIdx.x * bytes);
  const int64_t n = bytes / 16;
  uint32_t acc = 0;
  for (int64_t i = threadIdx.x; i < n; i += static_cast<int64_t>(blockDim.x) * U) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t j = i + static_cast<int64_t>(u) * blockDim.x;
      v[u] = j < n ? __ldcs(base + j) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc += v[u].x ^ v[u].w;
  }
  if (acc == 12345) *sink = acc;
}

static void run_ldg(int grid, int64_t per_cta, int64_t total, uint8_t* src, int* sink, cudaEvent_t e0, cudaEvent_t e1,
                    int U) {
  float best = 1e9f;
  for (int rep = 0; rep < 3; ++rep) {
    for (int w = 0; w < 6; ++w) {
      if (U == 8) probe_ldg<8><<<grid, 256>>>(src + w * total, per_cta, sink);
      else probe_ldg<16><<<grid, 256>>>(src + w * total, per_cta, sink);
    }
    cudaEventRecord(e0);
    for (int w = 0; w < 12; ++w) {
      if (U == 8) probe_ldg<8><<<grid, 256>>>(src + (w % 6) * total, per_cta, sink);
      else probe_ldg<16><<<grid, 256>>>(src + (w % 6) * total, per_cta, sink);
    }
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= 12;
    if (ms < best) best = ms;
  }
  const double gbs = static_cast<double>(per_cta) * grid / (best * 1e-3) / 1e9;
  printf("ldg grid %d U %d (%d KB in flight): %.2f us %.0f GB/s\n", grid, U, 256 * 16 * U / 1024, best * 1e3, gbs);
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int64_t per_cta = 640 * 1024;
  const int64_t total = per_cta * 160;  // one buffer; 6 rotate (600 MB >> L2, clean lines only)
  uint8_t* src;
  int* sink;
  cudaMalloc(&src, total * 6);
  cudaMalloc(&sink, 4);
  cudaMemset(src, 1, total * 6);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  printf("grid slot_KB chunk_KB slots inflight_KB  us   GB/s_total  GB/s_per_SM\n");
  const int grids[] = {128, 148};
  const int cfg[][3] = {{8, 8, 22}, {8, 8, 26}, {24, 24, 7}, {24, 8, 7}, {24, 4, 7}, {16, 16, 12}, {32, 32, 6}, {8, 2, 22}, {4, 4, 50}};
  for (int gi = 0; gi < 2; ++gi)
    for (const auto& c : cfg) {
      const int B = c[0] * 1024, ch = c[1] * 1024, S = c[2];
      const size_t smem = static_cast<size_t>(S) * B + 2 * S * 8;
      if (smem > 227 * 1024) continue;
      const int64_t bytes = per_cta / B * B;
      float best = 1e9f;
      for (int rep = 0; rep < 3; ++rep) {
        for (int w = 0; w < 6; ++w) probe<<<grids[gi], 64, smem>>>(src + w * total, bytes, S, B, ch, sink);
        cudaEventRecord(e0);
        for (int w = 0; w < 12; ++w) probe<<<grids[gi], 64, smem>>>(src + (w % 6) * total, bytes, S, B, ch, sink);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        ms /= 12;
        if (ms < best) best = ms;
      }
      const double gbs = static_cast<double>(bytes) * grids[gi] / (best * 1e-3) / 1e9;
      printf("%4d %7d %8d %5d %11d %6.2f %10.0f %11.1f\n", grids[gi], c[0], c[1], S, c[0] * S, best * 1e3, gbs,
             gbs / grids[gi]);
    }
  // B: producer lanes
  cudaFuncSetAttribute(probe_lanes, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  const int lcfg[][3] = {{8, 24, 1}, {8, 24, 2}, {8, 24, 4}, {8, 24, 8}, {16, 12, 4}, {4, 48, 8}};
  for (const auto& c : lcfg) {
    const int B = c[0] * 1024, S = c[1], P = c[2];
    const size_t smem = static_cast<size_t>(S) * B + 2 * S * 8;
    const int64_t bytes = per_cta / B * B;
    float best = 1e9f;
    for (int rep = 0; rep < 3; ++rep) {
      for (int w = 0; w < 6; ++w) probe_lanes<<<148, 64, smem>>>(src + w * total, bytes, S, B, P, sink);
      cudaEventRecord(e0);
      for (int w = 0; w < 12; ++w) probe_lanes<<<148, 64, smem>>>(src + (w % 6) * total, bytes, S, B, P, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      ms /= 12;
      if (ms < best) best = ms;
    }
    const double gbs = static_cast<double>(bytes) * 148 / (best * 1e-3) / 1e9;
    printf("lanes: slot %d KB x %d slots, %d producer lanes: %.2f us %.0f GB/s\n", c[0], S, P, best * 1e3, gbs);
  }
  run_ldg(148, per_cta, total, src, sink, e0, e1, 8);
  run_ldg(148, per_cta, total, src, sink, e0, e1, 16);
  run_ldg(296, per_cta / 2, total, src, sink, e0, e1, 8);
  cudaError_t err = cudaDeviceSynchronize();
  printf("status: %s (SMs %d)\n", cudaGetErrorString(err), nsm);
  return 0;
}
