// Shared tcgen05 helpers of the tensor-core triplet kernels (triplet_tc.cu,
// triplet_tc_bwd.cu): mbarriers, UMMA descriptors (K-major SWIZZLE_128B), the
// 3xTF32 split and the shared-memory operand writer.
#pragma once

#include <cstdint>

namespace egn {
namespace tc {

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c));
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(
          su32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* b) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ uint64_t kdesc(uint32_t saddr) {
  return static_cast<uint64_t>((saddr >> 4) & 0x3FFF) | (static_cast<uint64_t>(1) << 16) |
         (static_cast<uint64_t>(1024 >> 4) << 32) | (static_cast<uint64_t>(1) << 46) | (static_cast<uint64_t>(2) << 61);
}
__device__ __forceinline__ void mma_tf32(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.b32 %0, 1, 0, P;\n\t}" : "=r"(pred));
  return pred != 0;
}
__device__ __forceinline__ float tf32_rna(float x) { return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xffffe000u); }
__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// 16-byte granule g (0..7) of row r in a K-major SWIZZLE_128B slab (128 B rows, 8-row atoms)
__device__ __forceinline__ int sw_off(int r, int g) { return r * 128 + ((g ^ (r & 7)) << 4); }

// write 8 consecutive k values (k-step j of the slab) of row r as hi and lo
__device__ __forceinline__ void put8(uint8_t* hi, uint8_t* lo, int r, int j, const float* v) {
  float h[8], l[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    h[i] = tf32_rna(v[i]);
    l[i] = v[i] - h[i];
  }
  *reinterpret_cast<float4*>(hi + sw_off(r, 2 * j)) = make_float4(h[0], h[1], h[2], h[3]);
  *reinterpret_cast<float4*>(hi + sw_off(r, 2 * j + 1)) = make_float4(h[4], h[5], h[6], h[7]);
  *reinterpret_cast<float4*>(lo + sw_off(r, 2 * j)) = make_float4(l[0], l[1], l[2], l[3]);
  *reinterpret_cast<float4*>(lo + sw_off(r, 2 * j + 1)) = make_float4(l[4], l[5], l[6], l[7]);
}

}  // namespace tc
}  // namespace egn
