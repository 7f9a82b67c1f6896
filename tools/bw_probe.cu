// bw_probe.cu — HBM streaming probes (diagnostic, not product): how fast can one CTA per SM stream
// contiguous rows with (a) 1-D bulk copies into an mbarrier ring, (b) the same + a consumer that reads
// the smem rows, (c) plain LDG.128 with many loads in flight.  nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c)); }
__device__ __forceinline__ void expect_tx(uint64_t* b, uint32_t n) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory"); }
__device__ __forceinline__ void arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory"); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}" ::"r"(su32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void bulk(void* d, const void* s, uint32_t n, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(d)), "l"(s), "r"(n), "r"(su32(b)) : "memory");
}

template <int READ>
__global__ void __launch_bounds__(288, 1) ring_kernel(const uint8_t* W, size_t total, int rowbytes, int nslot, float* sink) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + (size_t)nslot * rowbytes);
  uint64_t* empty = full + nslot;
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const size_t nrows = total / rowbytes;
  const size_t r0 = nrows * blockIdx.x / gridDim.x, r1 = nrows * (blockIdx.x + 1) / gridDim.x;
  if (tid == 0) {
    for (int i = 0; i < nslot; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 8); }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (warp == 8) {
    if (lane == 0)
      for (size_t i = 0; i < r1 - r0; ++i) {
        int s = i % nslot;
        wait(&empty[s], ((i / nslot) & 1) ^ 1);
        expect_tx(&full[s], rowbytes);
        bulk(sm + (size_t)s * rowbytes, W + (r0 + i) * rowbytes, rowbytes, &full[s]);
      }
    return;
  }
  float acc = 0.f;
  for (size_t i = 0; i < r1 - r0; ++i) {
    int s = i % nslot;
    wait(&full[s], (i / nslot) & 1);
    if (READ) {
      const float4* row = reinterpret_cast<const float4*>(sm + (size_t)s * rowbytes);
      for (int c = warp * 32 + lane; c < rowbytes / 16; c += 256) { float4 v = row[c]; acc += v.x + v.y + v.z + v.w; }
    }
    __syncwarp();
    if (lane == 0) arrive(&empty[s]);
  }
  if (acc == 123.f) sink[0] = acc;
}

__global__ void ldg_kernel(const uint4* W, size_t n16, float* sink) {
  float acc = 0.f;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 7 * stride < n16; i += 8 * stride) {
    uint4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(W + i + u * stride));
#pragma unroll
    for (int u = 0; u < 8; ++u) acc += __uint_as_float(v[u].x ^ v[u].y ^ v[u].z ^ v[u].w);
  }
  if (acc == 123.f) sink[0] = acc;
}

int main() {
  const size_t total = 2ull << 30;  // 2 GiB
  uint8_t* W;
  float* sink;
  cudaMalloc(&W, total);
  cudaMalloc(&sink, 4);
  cudaMemset(W, 1, total);
  int sms = 148;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto timeit = [&](auto launch, const char* name) {
    launch();
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("%-48s %8.1f GB/s  (%s)\n", name, 5.0 * total / (ms / 1e3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  };
  for (int rb : {8192, 16384, 32768, 65536}) {
    for (int ns : {2, 3, 4, 6, 8, 12}) {
      size_t smem = (size_t)ns * rb + 2 * ns * 8;
      if (smem > 227 * 1024) continue;
      cudaFuncSetAttribute(ring_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      cudaFuncSetAttribute(ring_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      char nm[96];
      snprintf(nm, 96, "bulk ring row=%d nslot=%d no-read", rb, ns);
      timeit([&] { ring_kernel<0><<<sms, 288, smem>>>(W, total, rb, ns, sink); }, nm);
      snprintf(nm, 96, "bulk ring row=%d nslot=%d read", rb, ns);
      timeit([&] { ring_kernel<1><<<sms, 288, smem>>>(W, total, rb, ns, sink); }, nm);
      if (2 * smem <= 227 * 1024) {  // two CTAs per SM, each with its own ring
        snprintf(nm, 96, "bulk ring row=%d nslot=%d read, 2 CTAs/SM", rb, ns);
        timeit([&] { ring_kernel<1><<<2 * sms, 288, smem>>>(W, total, rb, ns, sink); }, nm);
      }
    }
  }
  for (int bpsm : {2, 4, 8}) {
    char nm[96];
    snprintf(nm, 96, "ldg.128 x8 unroll, %d CTAs/SM x 256 thr", bpsm);
    timeit([&] { ldg_kernel<<<sms * bpsm, 256>>>(reinterpret_cast<const uint4*>(W), total / 16, sink); }, nm);
  }
  return 0;
}
