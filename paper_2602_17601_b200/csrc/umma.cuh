// tcgen05 (5th-generation tensor core) helpers for sm_100a: TMEM allocation,
// shared-memory matrix descriptors, kind::tf32 MMA, commit/mbarrier and
// TMEM -> register loads.  Raw PTX, no CUTLASS.
//
// Operand layout used throughout ("K-major, no swizzle"): an R x K operand
// (R = M rows of A or N rows of B, K = reduction) is stored as 8 x 4 core
// matrices of 128 contiguous bytes (8 rows x 16 B).  Element (r, k):
//
//     byte(r, k) = (r / 8) * SBO + (k / 4) * 128 + (r % 8) * 16 + (k % 4) * 4
//
// so LBO (the K-direction core-matrix stride) is 128 B and SBO (the stride
// between 8-row groups) is (KC / 4) * 128 B for a buffer holding KC columns
// of K.  One kind::tf32 MMA consumes K = 8, i.e. two core matrices along K:
// step s starts at base + s * 256 B.
//
// Precision: "3xTF32".  x = hi + lo with hi = rna_tf32(x) and lo = x - hi
// (exact in fp32); a.b ~= hi_a hi_b + hi_a lo_b + lo_a hi_b, each term on the
// tensor core with fp32 accumulation in TMEM: ~fp32 products (dropped term
// lo_a lo_b ~ 2^-22 relative), ~3x the work of plain TF32.
#pragma once

#include <stdint.h>

namespace umma {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ uint32_t kmajor_offset(int r, int k, uint32_t sbo) {
  return (uint32_t)(r >> 3) * sbo + (uint32_t)(k >> 2) * 128u + (uint32_t)(r & 7) * 16u +
         (uint32_t)(k & 3) * 4u;
}

// shared-memory matrix descriptor (tcgen05 "matrix descriptor"): start
// address, LBO, SBO in 16-byte units, version 1 (sm_100), SWIZZLE_NONE
__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}

// instruction descriptor, kind::tf32: D fp32, A/B tf32, both K-major, dense
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

// arrive on an mbarrier once every previously issued tcgen05.mma of this
// thread has completed (implies tcgen05.fence::before_thread_sync)
__device__ __forceinline__ void commit(uint64_t* mbar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(mbar))
               : "memory");
}

__device__ __forceinline__ void mbar_init(uint64_t* mbar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(mbar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* mbar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(smem_u32(mbar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// generic-proxy smem writes -> visible to the tensor core (async proxy)
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// TMEM allocation by one whole warp; the base address lands in *slot
template <int NCOLS>
__device__ __forceinline__ void tmem_alloc(uint32_t* slot) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(slot)),
               "n"(NCOLS)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
template <int NCOLS>
__device__ __forceinline__ void tmem_free(uint32_t base) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(base), "n"(NCOLS)
               : "memory");
}

// 32 lanes x 16 consecutive fp32 columns: thread t of the warp gets lane
// (warp % 4) * 32 + t, columns [col, col + 16).  taddr = base + (lane0 << 16) + col
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, "
      "[%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ float tf32_hi(float x) {
  uint32_t h;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(x));
  return __uint_as_float(h);
}

// x -> (hi, lo) at K-major position (r, k) of the hi and lo buffers
__device__ __forceinline__ void put_split(unsigned char* hi_buf, unsigned char* lo_buf, int r, int k,
                                          uint32_t sbo, float x) {
  const uint32_t o = kmajor_offset(r, k, sbo);
  const float h = tf32_hi(x);
  *(float*)(hi_buf + o) = h;
  *(float*)(lo_buf + o) = x - h;
}

// NX consecutive K positions k0 .. k0+NX-1 of operand row r (k0 = li * NX),
// split into hi / lo, with 16- / 8-byte stores (a warp over consecutive rows
// then writes whole 128-B core-matrix rows: no bank conflicts)
template <int NX>
__device__ __forceinline__ void putn_split(unsigned char* hb, unsigned char* lb, int r, int k0,
                                           uint32_t sbo, const float* x) {
  float h[NX], l[NX];
#pragma unroll
  for (int i = 0; i < NX; ++i) {
    h[i] = tf32_hi(x[i]);
    l[i] = x[i] - h[i];
  }
  const uint32_t base = (uint32_t)(r >> 3) * sbo + (uint32_t)(r & 7) * 16u + (uint32_t)(k0 >> 2) * 128u;
  if constexpr (NX == 6) {
    if ((k0 & 3) == 0) {
      *(float4*)(hb + base) = make_float4(h[0], h[1], h[2], h[3]);
      *(float2*)(hb + base + 128) = make_float2(h[4], h[5]);
      *(float4*)(lb + base) = make_float4(l[0], l[1], l[2], l[3]);
      *(float2*)(lb + base + 128) = make_float2(l[4], l[5]);
    } else {
      *(float2*)(hb + base + 8) = make_float2(h[0], h[1]);
      *(float4*)(hb + base + 128) = make_float4(h[2], h[3], h[4], h[5]);
      *(float2*)(lb + base + 8) = make_float2(l[0], l[1]);
      *(float4*)(lb + base + 128) = make_float4(l[2], l[3], l[4], l[5]);
    }
  } else if constexpr (NX == 4) {
    *(float4*)(hb + base) = make_float4(h[0], h[1], h[2], h[3]);
    *(float4*)(lb + base) = make_float4(l[0], l[1], l[2], l[3]);
  } else if constexpr (NX == 2) {
    *(float2*)(hb + base + (k0 & 3) * 4) = make_float2(h[0], h[1]);
    *(float2*)(lb + base + (k0 & 3) * 4) = make_float2(l[0], l[1]);
  } else {
#pragma unroll
    for (int i = 0; i < NX; ++i) {
      const uint32_t o = kmajor_offset(r, k0 + i, sbo);
      *(float*)(hb + o) = h[i];
      *(float*)(lb + o) = l[i];
    }
  }
}

// x = hi + lo (exact fp32) of NX consecutive K positions of operand row r
template <int NX>
__device__ __forceinline__ void getn(const unsigned char* hb, const unsigned char* lb, int r, int k0,
                                     uint32_t sbo, float* x) {
  const uint32_t base = (uint32_t)(r >> 3) * sbo + (uint32_t)(r & 7) * 16u + (uint32_t)(k0 >> 2) * 128u;
  if constexpr (NX == 6) {
    float4 a, b, c, d;
    float2 e, f;
    if ((k0 & 3) == 0) {
      a = *(const float4*)(hb + base);
      b = *(const float4*)(lb + base);
      e = *(const float2*)(hb + base + 128);
      f = *(const float2*)(lb + base + 128);
      x[0] = a.x + b.x; x[1] = a.y + b.y; x[2] = a.z + b.z; x[3] = a.w + b.w;
      x[4] = e.x + f.x; x[5] = e.y + f.y;
    } else {
      e = *(const float2*)(hb + base + 8);
      f = *(const float2*)(lb + base + 8);
      c = *(const float4*)(hb + base + 128);
      d = *(const float4*)(lb + base + 128);
      x[0] = e.x + f.x; x[1] = e.y + f.y;
      x[2] = c.x + d.x; x[3] = c.y + d.y; x[4] = c.z + d.z; x[5] = c.w + d.w;
    }
  } else if constexpr (NX == 4) {
    const float4 a = *(const float4*)(hb + base), b = *(const float4*)(lb + base);
    x[0] = a.x + b.x; x[1] = a.y + b.y; x[2] = a.z + b.z; x[3] = a.w + b.w;
  } else if constexpr (NX == 2) {
    const float2 a = *(const float2*)(hb + base + (k0 & 3) * 4), b = *(const float2*)(lb + base + (k0 & 3) * 4);
    x[0] = a.x + b.x; x[1] = a.y + b.y;
  } else {
#pragma unroll
    for (int i = 0; i < NX; ++i) {
      const uint32_t o = kmajor_offset(r, k0 + i, sbo);
      x[i] = *(const float*)(hb + o) + *(const float*)(lb + o);
    }
  }
}

// D[m][n] += sum_k A(m, k) B(n, k) over ksteps x 8 columns of K, 3xTF32.
// A and B buffers: K-major (see top), SBO sbo_a / sbo_b, 128-B LBO.
// Called by ONE thread.
__device__ __forceinline__ void gram_3xtf32(uint32_t tmem_d, const unsigned char* a_hi,
                                            const unsigned char* a_lo, uint32_t sbo_a,
                                            const unsigned char* b_hi, const unsigned char* b_lo,
                                            uint32_t sbo_b, int ksteps, uint32_t idesc,
                                            bool accumulate) {
  const uint32_t ah = smem_u32(a_hi), al = smem_u32(a_lo), bh = smem_u32(b_hi), bl = smem_u32(b_lo);
  for (int s = 0; s < ksteps; ++s) {
    const uint32_t off = (uint32_t)s * 256u;
    const uint64_t dah = desc(ah + off, 128, sbo_a), dal = desc(al + off, 128, sbo_a);
    const uint64_t dbh = desc(bh + off, 128, sbo_b), dbl = desc(bl + off, 128, sbo_b);
    mma_tf32(tmem_d, dal, dbh, idesc, (accumulate || s > 0) ? 1u : 0u);
    mma_tf32(tmem_d, dah, dbl, idesc, 1u);
    mma_tf32(tmem_d, dah, dbh, idesc, 1u);
  }
}

}  // namespace umma
