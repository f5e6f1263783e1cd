// Shared device helpers: complex fp64 on double2, the DMMA fp64 MMA wrapper
// (mma.sync m8n8k4 f64 -- sm_100a has no tcgen05 kind::f64, SURVEY.md
// finding 6), cp.async, and error plumbing for the C-ABI.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

#define KH_DEV __device__ __forceinline__
#define KH_HD __host__ __device__

// Device-side bounds checks of a checked build (-DKH_CHECKED, e.g.
// profiles/probes/checked_build.py): index and size invariants of the
// shared-memory staging and scatter paths; compiled out otherwise.
#ifdef KH_CHECKED
#include <cassert>
#define KH_ASSERT(cond) assert(cond)
#else
#define KH_ASSERT(cond) ((void)0)
#endif

// ---- complex fp64 -----------------------------------------------------------
KH_DEV double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
KH_DEV double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
KH_DEV double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
// a - b*c
KH_DEV double2 cfms(double2 a, double2 b, double2 c) {
  return make_double2(a.x - b.x * c.x + b.y * c.y, a.y - b.x * c.y - b.y * c.x);
}
KH_DEV double2 cinv(double2 a) {
  // One IEEE reciprocal instead of two divisions. Smith-style scaling is
  // unnecessary: pivots passing the reference's threshold check are O(1).
  const double r = __drcp_rn(a.x * a.x + a.y * a.y);  // == 1.0 / x, correctly rounded
  return make_double2(a.x * r, -a.y * r);
}
KH_DEV double cabs2(double2 a) { return a.x * a.x + a.y * a.y; }

// ---- DMMA ---------------------------------------------------------------------
// D(8x8) = A(8x4, row) * B(4x8, col) + C. Lane (g = lane>>2, t = lane&3):
// a = A[g][t], b = B[t][g], c/d = C[g][2t], C[g][2t+1].
// (not volatile: the compiler may interleave independent MMAs and loads)
KH_DEV void dmma884(double& d0, double& d1, double a, double b) {
  asm(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

// ---- cp.async -------------------------------------------------------------------
KH_DEV void cp_async8(void* smem, const void* gmem, bool valid) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  int sz = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
KH_DEV void cp_async16(void* smem, const void* gmem, bool valid) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  int sz = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
KH_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
KH_DEV void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// ---- bulk async copies (TMA engine, SASS UBLKCP) + mbarrier ------------------------
KH_DEV uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
KH_DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
// makes an initialized mbarrier visible to the async proxy (bulk copies)
KH_DEV void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }
KH_DEV void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
KH_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "KH_WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra KH_WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// global -> shared bulk copy of `bytes` (multiple of 16, both ends 16-byte
// aligned), completing as transaction bytes on `bar`
KH_DEV void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
