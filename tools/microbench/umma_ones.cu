// all-ones operands: D must be K (=128) everywhere for any layout / major mode
#include <cstdint>
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(layout) << 61;
  return d;
}
__global__ void k(float* dump, int variant) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* buf = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  const bool bf16 = variant & 4;
  for (int i = tid; i < 65536 / 4; i += 128)
    reinterpret_cast<uint32_t*>(buf)[i] = bf16 ? 0x3F803F80u : 0x3F800000u;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tbase)), "r"(128));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n");
  }
  asm volatile("fence.proxy.async.shared::cta;\n");
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tm = tbase;
  const int M = (variant & 8) ? 128 : 64, N = 64;
  const uint32_t major = (variant & 1) ? 1u : 0u;
  const uint32_t fmt = bf16 ? 1u : 2u;
  const uint32_t kind_bits = (1u << 4) | (fmt << 7) | (fmt << 10) | (major << 15) | (major << 16) |
                             (static_cast<uint32_t>(N >> 3) << 17) | (static_cast<uint32_t>(M >> 4) << 24);
  const uint32_t layout = (variant & 2) ? 2u : 0u;
  if (tid == 0) {
    for (int kk = 0; kk < 4; ++kk) {
      const uint64_t a = make_desc(smem_u32(buf) + kk * 1024, 128, 1024, layout);
      const uint64_t b = make_desc(smem_u32(buf) + 32768 + kk * 1024, 128, 1024, layout);
      const uint32_t acc = kk > 0;
      if (bf16)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tm), "l"(a), "l"(b), "r"(kind_bits), "r"(acc));
      else
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tm), "l"(a), "l"(b), "r"(kind_bits), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(&bar)));
    asm volatile("{\n\t.reg .pred P;\n\tW1:\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n\t@!P bra W1;\n\t}\n" ::"r"(smem_u32(&bar)));
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  uint32_t v[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "r"(tm + (static_cast<uint32_t>(warp * 32) << 16)));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n");
  for (int j = 0; j < 8; ++j) dump[tid * 8 + j] = __uint_as_float(v[j]);
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tm), "r"(128));
}
int main() {
  float* d;
  cudaMalloc(&d, 128 * 8 * 4);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 66 * 1024);
  for (int var = 0; var < 16; ++var) {
    cudaMemset(d, 0xFF, 128 * 8 * 4);
    k<<<1, 128, 66 * 1024>>>(d, var);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> h(128 * 8);
    cudaMemcpy(h.data(), d, h.size() * 4, cudaMemcpyDeviceToHost);
    printf("var %2d (%s M=%d %s %s): err=%s lanes0/16/31/32/64/100: %g %g %g %g %g %g\n", var, var & 4 ? "bf16" : "tf32",
           var & 8 ? 128 : 64, var & 1 ? "MN" : "K", var & 2 ? "SW128" : "none", cudaGetErrorString(e), h[0], h[16 * 8],
           h[31 * 8], h[32 * 8], h[64 * 8], h[100 * 8]);
    if (e != cudaSuccess) return 1;
  }
}
