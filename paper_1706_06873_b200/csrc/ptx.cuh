// ptx.cuh -- thin inline-PTX wrappers for sm_100a: mbarrier, TMA
// (cp.async.bulk.tensor), tcgen05 (alloc / mma / commit / ld) and the
// shared-memory / instruction descriptors the window GEMM uses.
// Written against the PTX ISA 8.7 instruction forms (CUDA 12.9).
#pragma once
#include <cstdint>

namespace mec {
namespace ptx {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ uint32_t lane_id() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%laneid;" : "=r"(r));
  return r;
}

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "elect.sync _|p, 0xffffffff;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(pred));
  return pred != 0;
}

// ------------------------------------------------------------ mbarrier
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Spin on try_wait without a suspend-time hint: with a hint ptxas emits
// NANOSLEEP.SYNCS between probes, whose wake-up latency showed up as the
// MMA <-> epilogue handshake bottleneck in ncu (tens of thousands of sleeps).
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(a),
      "r"(parity)
      : "memory");
}

// As mbar_wait, with cluster-scope acquire.  Not used on hot paths: a
// cluster-scope acquire makes ptxas emit an L1 invalidation (CCTL.IVALL) per
// probe -- the pair kernels' accumulator waits with it ran 20-60% slower (pair
// sweep cv4 b128 915 -> 1477 us).  The tcgen05 fences around the barrier
// order the TMEM accesses, as CUTLASS's cluster barriers do with plain waits.
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(a),
      "r"(parity)
      : "memory");
}

// try_wait with a nanosleep backoff between failed probes: for waits that are
// usually long (epilogue waiting for an accumulator, producer waiting for a
// slot), so idle warps do not keep the mbarrier unit busy.
__device__ __forceinline__ void mbar_wait_backoff(uint64_t* bar, uint32_t parity, uint32_t ns) {
  const uint32_t a = smem_u32(bar);
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, P1;\n\t}"
      : "=r"(ok)
      : "r"(a), "r"(parity)
      : "memory");
  while (!ok) {
    __nanosleep(ns);
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, P1;\n\t}"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
  }
}

// Pure spin on the non-blocking test_wait (no hardware suspend between probes).
__device__ __forceinline__ void mbar_spin(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "SPIN_%=:\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra SPIN_%=;\n\t}" ::"r"(a),
      "r"(parity)
      : "memory");
}

// ------------------------------------------------ programmatic dependent launch
// Primary kernel: let the next kernel on the stream start launching now.
__device__ __forceinline__ void griddep_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
// Dependent kernel: wait until the preceding kernel has completed and its
// memory operations are visible (a no-op when launched without PDL).
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// ------------------------------------------------------------------ TMA
__device__ __forceinline__ void tma_prefetch_desc(const void* desc) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(desc)) : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* smem_dst, const void* desc, uint64_t* bar,
                                            int32_t x, int32_t y, uint64_t cache_hint) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(desc)), "r"(smem_u32(bar)), "r"(x), "r"(y), "l"(cache_hint)
      : "memory");
}

__device__ __forceinline__ void tma_load_3d(void* smem_dst, const void* desc, uint64_t* bar,
                                            int32_t x, int32_t y, int32_t z, uint64_t cache_hint) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cta.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(desc)), "r"(smem_u32(bar)), "r"(x), "r"(y), "r"(z),
      "l"(cache_hint)
      : "memory");
}

// Non-tensor bulk copy global -> shared (16-byte aligned src/dst, size a
// multiple of 16), completing on an mbarrier (complete_tx::bytes).
__device__ __forceinline__ void bulk_load(void* smem_dst, const void* gsrc, uint32_t bytes,
                                          uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(gsrc)), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ uint32_t ld_shared_u32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ void st_shared_u32(uint32_t addr, uint32_t v) {
  asm volatile("st.shared.b32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}

// CTA-scope acquire load / release store of a shared-memory word (flags
// between warps of one CTA).
// relaxed gpu-scope load (a spin on a counter other CTAs bump; pair it with a fence)
__device__ __forceinline__ uint32_t ld_relaxed_gpu_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_acquire_shared_u32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_shared_u32(uint32_t addr, uint32_t v) {
  asm volatile("st.release.cta.shared::cta.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}

// Named barrier among `count` threads (id 1..15; 0 is __syncthreads).
__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// TMA stores (smem -> global, bulk-group completion), OOB rows/cols clipped.
__device__ __forceinline__ void tma_store_3d(const void* desc, const void* smem_src, int32_t x,
                                             int32_t y, int32_t z) {
  asm volatile(
      "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
          reinterpret_cast<uint64_t>(desc)),
      "r"(smem_u32(smem_src)), "r"(x), "r"(y), "r"(z)
      : "memory");
}
__device__ __forceinline__ void tma_store_4d(const void* desc, const void* smem_src, int32_t x,
                                             int32_t y, int32_t z, int32_t w) {
  asm volatile(
      "cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(
          reinterpret_cast<uint64_t>(desc)),
      "r"(smem_u32(smem_src)), "r"(x), "r"(y), "r"(z), "r"(w)
      : "memory");
}
__device__ __forceinline__ void bulk_commit_group() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
// Wait until at most N bulk groups are pending *reading* their smem source.
template <int N>
__device__ __forceinline__ void bulk_wait_group_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait_group() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c,
                                             uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c),
               "r"(d)
               : "memory");
}

__device__ __forceinline__ uint4 ld_shared_v4(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(addr)
               : "memory");
  return v;
}

__device__ __forceinline__ void tma_load_4d(void* smem_dst, const void* desc, uint64_t* bar,
                                            int32_t x, int32_t y, int32_t z, int32_t w,
                                            uint64_t cache_hint) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cta.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4, %5, %6}], [%2], %7;" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(desc)), "r"(smem_u32(bar)), "r"(x), "r"(y), "r"(z), "r"(w),
      "l"(cache_hint)
      : "memory");
}

// L2 cache-policy descriptors for the .L2::cache_hint operand
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// -------------------------------------------------------------- tcgen05
template <uint32_t kCols>
__device__ __forceinline__ void tmem_alloc(uint32_t* smem_result) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(smem_result)),
               "n"(kCols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void tmem_alloc_dyn(uint32_t* smem_result, uint32_t cols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(smem_result)),
               "r"(cols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t cols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(cols)
               : "memory");
}

__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// D[tmem] (+)= A[smem] * B[smem]^T, both K-major; kind::f16 (bf16) or kind::tf32.
template <bool kTF32>
__device__ __forceinline__ void mma_ss(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                       uint32_t idesc, uint32_t accumulate) {
  if constexpr (kTF32) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
  } else {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
  }
}

// Same, executed by a whole warp with warp-uniform operands: one elected lane
// issues the MMA (descriptor arithmetic stays on the uniform datapath).
template <bool kTF32>
__device__ __forceinline__ void mma_ss_elect(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                             uint32_t idesc, uint32_t accumulate) {
  if constexpr (kTF32) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
  } else {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
  }
}

// Whole-warp call, A operand in tensor memory ("TS" form): D[tmem] (+)= A[tmem] B[smem].
// A is M x K with row m in TMEM lane m, K packed along 32-bit columns
// (2 bf16 or 1 tf32 per column); a_tmem addresses the MMA's first column.
template <bool kTF32>
__device__ __forceinline__ void mma_ts_elect(uint32_t tmem_d, uint32_t a_tmem, uint64_t bdesc,
                                             uint32_t idesc, uint32_t accumulate) {
  if constexpr (kTF32) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
        "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
  } else {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
        "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
  }
}

// Whole-warp call: one elected lane issues the 4 SS MMAs of a 128-byte K atom
// (A and B descriptors + 0/2/4/6 in 16-byte units, i.e. 32-byte K steps).
// accumulate applies to the first MMA; the other three always accumulate.
template <bool kTF32>
__device__ __forceinline__ void mma_ss_atom_elect(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                                  uint32_t idesc, uint32_t accumulate) {
  if constexpr (kTF32) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t.reg .b64 a1, a2, a3, b1, b2, b3;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "add.u64 a1, %1, 2;\n\tadd.u64 a2, %1, 4;\n\tadd.u64 a3, %1, 6;\n\t"
        "add.u64 b1, %2, 2;\n\tadd.u64 b2, %2, 4;\n\tadd.u64 b3, %2, 6;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], a1, b1, %3, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], a2, b2, %3, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], a3, b3, %3, 1;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
  } else {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t.reg .b64 a1, a2, a3, b1, b2, b3;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "add.u64 a1, %1, 2;\n\tadd.u64 a2, %1, 4;\n\tadd.u64 a3, %1, 6;\n\t"
        "add.u64 b1, %2, 2;\n\tadd.u64 b2, %2, 4;\n\tadd.u64 b3, %2, 6;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a1, b1, %3, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a2, b2, %3, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a3, b3, %3, 1;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
  }
}

// As mma_ss_atom_elect, with an independent B descriptor per 32-byte K step
// (multi-row tiles whose window shift is a whole K step but not a whole atom).
template <bool kTF32>
__device__ __forceinline__ void mma_ss_atom4b_elect(uint32_t tmem_d, uint64_t adesc, uint64_t b0, uint64_t b1,
                                                    uint64_t b2, uint64_t b3, uint32_t idesc,
                                                    uint32_t accumulate) {
  if constexpr (kTF32) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t.reg .b64 a1, a2, a3;\n\t"
        "setp.ne.b32 p, %7, 0;\n\t"
        "add.u64 a1, %1, 2;\n\tadd.u64 a2, %1, 4;\n\tadd.u64 a3, %1, 6;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %6, p;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], a1, %3, %6, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], a2, %4, %6, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], a3, %5, %6, 1;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(b0), "l"(b1), "l"(b2), "l"(b3), "r"(idesc), "r"(accumulate)
        : "memory");
  } else {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t.reg .b64 a1, a2, a3;\n\t"
        "setp.ne.b32 p, %7, 0;\n\t"
        "add.u64 a1, %1, 2;\n\tadd.u64 a2, %1, 4;\n\tadd.u64 a3, %1, 6;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %6, p;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a1, %3, %6, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a2, %4, %6, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a3, %5, %6, 1;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(b0), "l"(b1), "l"(b2), "l"(b3), "r"(idesc), "r"(accumulate)
        : "memory");
  }
}

// Whole-warp call: one elected lane issues the 4 TS MMAs of a 128-byte A atom
// (K = 4 x 32 bytes: A columns a_tmem + 0/8/16/24, B descriptor + 0/2/4/6 in
// 16-byte units) -- one election and one operand transfer per atom.
// accumulate applies to the first MMA; the other three always accumulate.
template <bool kTF32>
__device__ __forceinline__ void mma_ts_atom_elect(uint32_t tmem_d, uint32_t a_tmem, uint64_t bdesc,
                                                  uint32_t idesc, uint32_t accumulate) {
  if constexpr (kTF32) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t.reg .b32 a1, a2, a3;\n\t.reg .b64 b1, b2, b3;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "add.u32 a1, %1, 8;\n\tadd.u32 a2, %1, 16;\n\tadd.u32 a3, %1, 24;\n\t"
        "add.u64 b1, %2, 2;\n\tadd.u64 b2, %2, 4;\n\tadd.u64 b3, %2, 6;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [a1], b1, %3, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [a2], b2, %3, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [a3], b3, %3, 1;\n\t}" ::"r"(tmem_d),
        "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
  } else {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t.reg .b32 a1, a2, a3;\n\t.reg .b64 b1, b2, b3;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "add.u32 a1, %1, 8;\n\tadd.u32 a2, %1, 16;\n\tadd.u32 a3, %1, 24;\n\t"
        "add.u64 b1, %2, 2;\n\tadd.u64 b2, %2, 4;\n\tadd.u64 b3, %2, 6;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a1], b1, %3, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a2], b2, %3, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a3], b3, %3, 1;\n\t}" ::"r"(tmem_d),
        "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
  }
}

// Whole-warp call: one elected lane issues the first n (1..4) of the 4 TS
// MMAs of a 128-byte K group: A columns a_tmem + 0/8/16/24, B descriptor
// + 0/2/4/6 (16-byte units, i.e. 32-byte K steps).  accumulate applies to the
// first MMA; the others always accumulate.
template <bool kTF32>
__device__ __forceinline__ void mma_ts_grp_elect(uint32_t tmem_d, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc,
                                                 uint32_t accumulate, int n) {
#define MEC_TS_GRP_BODY(KIND)                                                                 \
  asm volatile(                                                                               \
      "{\n\t.reg .pred p, e, e1, e2, e3;\n\t.reg .b32 a1, a2, a3;\n\t.reg .b64 b1, b2, b3;\n\t"    \
      "setp.ne.b32 p, %4, 0;\n\t"                                                             \
      "add.u32 a1, %1, 8;\n\tadd.u32 a2, %1, 16;\n\tadd.u32 a3, %1, 24;\n\t"                    \
      "add.u64 b1, %2, 2;\n\tadd.u64 b2, %2, 4;\n\tadd.u64 b3, %2, 6;\n\t"                      \
      "elect.sync _|e, 0xffffffff;\n\t"                                                       \
      "setp.gt.and.s32 e1, %5, 1, e;\n\t"                                                     \
      "setp.gt.and.s32 e2, %5, 2, e;\n\t"                                                     \
      "setp.gt.and.s32 e3, %5, 3, e;\n\t"                                                     \
      "@e tcgen05.mma.cta_group::1.kind::" KIND " [%0], [%1], %2, %3, p;\n\t"                   \
      "@e1 tcgen05.mma.cta_group::1.kind::" KIND " [%0], [a1], b1, %3, 1;\n\t"                  \
      "@e2 tcgen05.mma.cta_group::1.kind::" KIND " [%0], [a2], b2, %3, 1;\n\t"                  \
      "@e3 tcgen05.mma.cta_group::1.kind::" KIND " [%0], [a3], b3, %3, 1;\n\t}" ::"r"(tmem_d),  \
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate), "r"(n)                             \
      : "memory")
  if constexpr (kTF32) {
    MEC_TS_GRP_BODY("tf32");
  } else {
    MEC_TS_GRP_BODY("f16");
  }
#undef MEC_TS_GRP_BODY
}

// Whole-warp call: the 4 TS MMAs of a 128-byte K group (A columns a_tmem +
// 0/8/16/24, B descriptor low word + 0/2/4/6; the high word is the constant
// of smem_desc_sw128), issued by one elected lane behind a branch rather than
// per-instruction predicates (fewer uniform-register moves per MMA).
template <bool kTF32>
__device__ __forceinline__ void mma_ts_atom_br(uint32_t tmem_d, uint32_t a_tmem, uint32_t bdesc_lo, uint32_t idesc,
                                               uint32_t accumulate) {
#define MEC_TS_BR_BODY(KIND)                                                                         \
  asm volatile(                                                                                      \
      "{\n\t.reg .pred p, e;\n\t.reg .b32 a1, a2, a3, l1, l2, l3;\n\t.reg .b64 b0, b1, b2, b3;\n\t"       \
      "elect.sync _|e, 0xffffffff;\n\t"                                                              \
      "@!e bra SKIP_%=;\n\t"                                                                         \
      "setp.ne.b32 p, %4, 0;\n\t"                                                                    \
      "add.u32 a1, %1, 8;\n\tadd.u32 a2, %1, 16;\n\tadd.u32 a3, %1, 24;\n\t"                           \
      "add.u32 l1, %2, 2;\n\tadd.u32 l2, %2, 4;\n\tadd.u32 l3, %2, 6;\n\t"                             \
      "mov.b64 b0, {%2, 0x40004040};\n\tmov.b64 b1, {l1, 0x40004040};\n\t"                             \
      "mov.b64 b2, {l2, 0x40004040};\n\tmov.b64 b3, {l3, 0x40004040};\n\t"                             \
      "tcgen05.mma.cta_group::1.kind::" KIND " [%0], [%1], b0, %3, p;\n\t"                             \
      "tcgen05.mma.cta_group::1.kind::" KIND " [%0], [a1], b1, %3, 1;\n\t"                             \
      "tcgen05.mma.cta_group::1.kind::" KIND " [%0], [a2], b2, %3, 1;\n\t"                             \
      "tcgen05.mma.cta_group::1.kind::" KIND " [%0], [a3], b3, %3, 1;\n\t"                             \
      "SKIP_%=:\n\t}" ::"r"(tmem_d),                                                                  \
      "r"(a_tmem), "r"(bdesc_lo), "r"(idesc), "r"(accumulate)                                        \
      : "memory")
  if constexpr (kTF32) {
    MEC_TS_BR_BODY("tf32");
  } else {
    MEC_TS_BR_BODY("f16");
  }
#undef MEC_TS_BR_BODY
}

// Whole-warp call: one elected lane issues n_groups (>= 1) consecutive
// 128-byte K groups of TS MMAs into one accumulator, in a PTX loop (no
// per-group election or convergence code): group g reads A at TMEM column
// a_tmem + 32 g (wrapping from ring_end back by ring_cols), steps + 0/8/16/24,
// and B at descriptor low word b_lo + g b_step + 0/2/4/6 (high word: the
// constant of smem_desc_sw128).  The first MMA accumulates iff accumulate.
template <bool kTF32>
__device__ __forceinline__ void mma_ts_groups_elect(uint32_t tmem_d, uint32_t a_tmem, uint32_t ring_end,
                                                    uint32_t ring_cols, uint32_t b_lo, uint32_t b_step,
                                                    uint32_t idesc, uint32_t accumulate, int n_groups) {
#define MEC_TS_LOOP_BODY(KIND)                                                                         \
  asm volatile(                                                                                        \
      "{\n\t.reg .pred e, p, w, more;\n\t.reg .b32 c, b, g, a1, a2, a3, l1, l2, l3, hi;\n\t"             \
      ".reg .b64 b0, b1, b2, b3;\n\t"                                                                  \
      "elect.sync _|e, 0xffffffff;\n\t"                                                                \
      "@!e bra DONE_%=;\n\t"                                                                           \
      "mov.b32 hi, 0x40004040;\n\t"                                                                    \
      "mov.b32 c, %1;\n\tmov.b32 b, %4;\n\tmov.b32 g, 0;\n\t"                                           \
      "setp.ne.b32 p, %7, 0;\n"                                                                        \
      "LOOP_%=:\n\t"                                                                                   \
      "add.u32 a1, c, 8;\n\tadd.u32 a2, c, 16;\n\tadd.u32 a3, c, 24;\n\t"                                \
      "add.u32 l1, b, 2;\n\tadd.u32 l2, b, 4;\n\tadd.u32 l3, b, 6;\n\t"                                  \
      "mov.b64 b0, {b, hi};\n\tmov.b64 b1, {l1, hi};\n\tmov.b64 b2, {l2, hi};\n\tmov.b64 b3, {l3, hi};\n\t" \
      "tcgen05.mma.cta_group::1.kind::" KIND " [%0], [c], b0, %6, p;\n\t"                        \
      "tcgen05.mma.cta_group::1.kind::" KIND " [%0], [a1], b1, %6, 1;\n\t"                       \
      "tcgen05.mma.cta_group::1.kind::" KIND " [%0], [a2], b2, %6, 1;\n\t"                       \
      "tcgen05.mma.cta_group::1.kind::" KIND " [%0], [a3], b3, %6, 1;\n\t"                       \
      "setp.ne.b32 p, 1, 0;\n\t"                                                                       \
      "add.u32 c, c, 32;\n\tsetp.ge.u32 w, c, %2;\n\t@w sub.u32 c, c, %3;\n\t"                          \
      "add.u32 b, b, %5;\n\tadd.u32 g, g, 1;\n\t"                                                      \
      "setp.lt.s32 more, g, %8;\n\t@more bra LOOP_%=;\n"                                                \
      "DONE_%=:\n\t}" ::"r"(tmem_d),                                                                   \
      "r"(a_tmem), "r"(ring_end), "r"(ring_cols), "r"(b_lo), "r"(b_step), "r"(idesc), "r"(accumulate),    \
      "r"(n_groups)                                                                                     \
      : "memory")
  if constexpr (kTF32) {
    MEC_TS_LOOP_BODY("tf32");
  } else {
    MEC_TS_LOOP_BODY("f16");
  }
#undef MEC_TS_LOOP_BODY
}

// Whole-warp call: one elected lane issues a whole row of n_groups (>= 1)
// 128-byte K groups of TS MMAs (as mma_ts_groups_elect), waiting inside the
// same PTX loop for every A atom a group needs: group g ends at stream element
// a + ((g + 1) << grp_log2) - 1, held by atom >> bkl; atoms are waited in
// ring order on the mbarriers afull_base + 8 slot (phase parity wphase),
// starting from ring slot wslot with `avail` atoms already landed.  The
// caller advances its own copy of (wslot, wphase, avail) past the last atom
// the row needs (the elected lane's counters are not returned).  One call per
// row: no per-group or per-run control code in the warp (latency-bound).
#ifndef MEC_PAIR_WAITSEM
#define MEC_PAIR_WAITSEM ".acquire.cluster"
#endif
template <bool kTF32, bool kPair = false>
__device__ __forceinline__ void mma_ts_row_elect(uint32_t tmem_d, uint32_t a_tmem, uint32_t ring_end,
                                                 uint32_t ring_cols, uint32_t b_lo, uint32_t b_step,
                                                 uint32_t idesc, int n_groups, int a, int grp_log2, int bkl,
                                                 uint32_t afull_base, int wslot, uint32_t wphase, int avail,
                                                 int ns) {
#define MEC_TS_ROW_BODY(KIND, GRP, WAITSEM)                                                            \
  asm volatile(                                                                                        \
      "{\n\t.reg .pred e, p, w, more, ok, fin;\n\t"                                                    \
      ".reg .b32 c, b, g, a1, a2, a3, l1, l2, l3, hi, need, t, ws, wp, av, bar;\n\t"                    \
      ".reg .b64 b0, b1, b2, b3;\n\t"                                                                  \
      "elect.sync _|e, 0xffffffff;\n\t"                                                                \
      "@!e bra DONE_%=;\n\t"                                                                           \
      "mov.b32 hi, 0x40004040;\n\t"                                                                    \
      "mov.b32 c, %1;\n\tmov.b32 b, %4;\n\tmov.b32 g, 0;\n\t"                                           \
      "mov.b32 ws, %12;\n\tmov.b32 wp, %13;\n\tmov.b32 av, %14;\n\t"                                     \
      "setp.ne.b32 p, 0, 0;\n"                                                                         \
      "LOOP_%=:\n\t"                                                                                   \
      "add.u32 t, g, 1;\n\tshl.b32 t, t, %10;\n\tadd.u32 t, t, %9;\n\tsub.u32 t, t, 1;\n\t"               \
      "shr.s32 need, t, %11;\n"                                                                        \
      "WAIT_%=:\n\t"                                                                                   \
      "setp.gt.s32 ok, av, need;\n\t@ok bra READY_%=;\n\t"                                              \
      "mad.lo.u32 bar, ws, 8, %15;\n"                                                                  \
      "SPIN_%=:\n\t"                                                                                   \
      "mbarrier.try_wait.parity" WAITSEM ".shared::cta.b64 w, [bar], wp;\n\t"                           \
      "@!w bra SPIN_%=;\n\t"                                                                           \
      "add.u32 ws, ws, 1;\n\tsetp.eq.u32 fin, ws, %16;\n\t@fin mov.b32 ws, 0;\n\t@fin xor.b32 wp, wp, 1;\n\t" \
      "add.u32 av, av, 1;\n\tbra WAIT_%=;\n"                                                            \
      "READY_%=:\n\t"                                                                                  \
      "tcgen05.fence::after_thread_sync;\n\t"                                                          \
      "add.u32 a1, c, 8;\n\tadd.u32 a2, c, 16;\n\tadd.u32 a3, c, 24;\n\t"                                \
      "add.u32 l1, b, 2;\n\tadd.u32 l2, b, 4;\n\tadd.u32 l3, b, 6;\n\t"                                  \
      "mov.b64 b0, {b, hi};\n\tmov.b64 b1, {l1, hi};\n\tmov.b64 b2, {l2, hi};\n\tmov.b64 b3, {l3, hi};\n\t" \
      "tcgen05.mma.cta_group::" GRP ".kind::" KIND " [%0], [c], b0, %6, p;\n\t"                        \
      "tcgen05.mma.cta_group::" GRP ".kind::" KIND " [%0], [a1], b1, %6, 1;\n\t"                       \
      "tcgen05.mma.cta_group::" GRP ".kind::" KIND " [%0], [a2], b2, %6, 1;\n\t"                       \
      "tcgen05.mma.cta_group::" GRP ".kind::" KIND " [%0], [a3], b3, %6, 1;\n\t"                       \
      "setp.ne.b32 p, 1, 0;\n\t"                                                                       \
      "add.u32 c, c, 32;\n\tsetp.ge.u32 w, c, %2;\n\t@w sub.u32 c, c, %3;\n\t"                          \
      "add.u32 b, b, %5;\n\tadd.u32 g, g, 1;\n\t"                                                      \
      "setp.lt.s32 more, g, %7;\n\t@more bra LOOP_%=;\n"                                                \
      "DONE_%=:\n\t}" ::"r"(tmem_d),                                                                   \
      "r"(a_tmem), "r"(ring_end), "r"(ring_cols), "r"(b_lo), "r"(b_step), "r"(idesc), "r"(n_groups),      \
      "r"(0), "r"(a), "r"(grp_log2), "r"(bkl), "r"(wslot), "r"(wphase), "r"(avail), "r"(afull_base),   \
      "r"(ns)                                                                                          \
      : "memory")
  // kPair: the CTA pair's MMA (cta_group::2, M = 256; A from both CTAs' TMEM
  // at the same columns) and cluster-scope acquire on the ring barriers, which
  // the peer CTA's copiers arrive on remotely
  if constexpr (kPair) {
    if constexpr (kTF32) {
      MEC_TS_ROW_BODY("tf32", "2", MEC_PAIR_WAITSEM);
    } else {
      MEC_TS_ROW_BODY("f16", "2", MEC_PAIR_WAITSEM);
    }
  } else {
    if constexpr (kTF32) {
      MEC_TS_ROW_BODY("tf32", "1", "");
    } else {
      MEC_TS_ROW_BODY("f16", "1", "");
    }
  }
#undef MEC_TS_ROW_BODY
}

// Whole-warp call: one elected lane copies a 128-row x 128-byte SW128 K-major
// atom from shared memory (descriptor sdesc) into TMEM columns taddr ..
// taddr + 31 (row m -> lane m, 2 bf16 / 1 fp32 per 32-bit column): 4 x
// tcgen05.cp.128x256b of its 32-byte K chunks (descriptor start + 32 B each).
// Copies and MMAs issued by one thread execute in issue order.
__device__ __forceinline__ void tmem_cp_atom_elect(uint32_t taddr, uint64_t sdesc) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t.reg .b64 d1, d2, d3;\n\t.reg .b32 t1, t2, t3;\n\t"
      "add.u64 d1, %1, 2;\n\tadd.u64 d2, %1, 4;\n\tadd.u64 d3, %1, 6;\n\t"
      "add.u32 t1, %0, 8;\n\tadd.u32 t2, %0, 16;\n\tadd.u32 t3, %0, 24;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.cp.cta_group::1.128x256b [%0], %1;\n\t"
      "@e tcgen05.cp.cta_group::1.128x256b [t1], d1;\n\t"
      "@e tcgen05.cp.cta_group::1.128x256b [t2], d2;\n\t"
      "@e tcgen05.cp.cta_group::1.128x256b [t3], d3;\n\t}" ::"r"(taddr),
      "l"(sdesc)
      : "memory");
}

// Whole-warp call: one elected lane commits (arrives on `bar` when done).
__device__ __forceinline__ void mma_commit_elect(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(
          smem_u32(bar))
      : "memory");
}

// All previously issued tcgen05.mma of this thread arrive on `bar` when done.
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

// 32 lanes x 32-bit, 16 consecutive columns: thread t of the warp gets row
// (lane_base + t), columns [col, col+16).
__device__ __forceinline__ void tmem_ld_32x32b_x16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}

// Warp-wide store of 32 consecutive 32-bit columns: lane i writes TMEM lane
// (taddr lane base + i), register j -> column (taddr column + j).
__device__ __forceinline__ void tmem_st_32x32b_x32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, "
      "%17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]),
      "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]),
      "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}

__device__ __forceinline__ void tmem_st_32x32b_x16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}

__device__ __forceinline__ void tmem_st_32x32b_x4(uint32_t taddr, uint32_t r0, uint32_t r1, uint32_t r2,
                                                  uint32_t r3) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(taddr), "r"(r0), "r"(r1),
               "r"(r2), "r"(r3)
               : "memory");
}

__device__ __forceinline__ void tmem_st_wait() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ uint2 ld_shared_v2(uint32_t addr) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(addr));
  return v;
}

__device__ __forceinline__ void tmem_ld_wait() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}


// ------------------------------------------------ CTA pairs (cta_group::2)
// A cluster of 2 CTAs on the two SMs of a TPC issues tcgen05 work as one
// "CTA pair": the leader (rank 0) issues the MMAs, whose M =
// 256 rows come 128 from each CTA's shared memory (A) and whose N columns of B
// are split N/2 per CTA; each CTA's TMEM receives its 128 rows of D.
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_id_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t nclusters_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
  return r;
}
// shared::cluster address of the same shared variable in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa_shared(uint32_t smem_addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// arrive on an mbarrier given by its shared::cluster address (possibly the peer CTA's)
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// TMA load into this CTA's shared memory whose completion (complete_tx) is
// signalled on the mbarrier at shared::cluster address `bar_cluster` -- the
// pair leader's barrier, so one expect_tx there covers both CTAs' loads.
__device__ __forceinline__ void tma_load_2d_pair(void* smem_dst, const void* desc, uint32_t bar_cluster, int32_t x,
                                                 int32_t y, uint64_t cache_hint) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(desc)), "r"(bar_cluster), "r"(x), "r"(y), "l"(cache_hint)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d_pair(void* smem_dst, const void* desc, uint32_t bar_cluster, int32_t x,
                                                 int32_t y, int32_t z, uint64_t cache_hint) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(desc)), "r"(bar_cluster), "r"(x), "r"(y), "r"(z), "l"(cache_hint)
      : "memory");
}
// As tma_load_2d_pair, multicast to the CTAs of cta_mask (same shared offset in
// each); bar_cta is this CTA's own (shared::cta) address of the barrier, with
// the pair bit cleared so each destination pair's LEADER barrier counts the
// bytes (the CUTLASS SM100 2-SM multicast convention).
__device__ __forceinline__ void tma_load_2d_pair_mc(void* smem_dst, const void* desc, uint32_t bar_cta, uint16_t cta_mask,
                                                    int32_t x, int32_t y, uint64_t cache_hint) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      ".L2::cache_hint [%0], [%1, {%4, %5}], [%2], %3, %6;" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(desc)), "r"(bar_cta & 0xFEFFFFFFu), "h"(cta_mask), "r"(x), "r"(y),
      "l"(cache_hint)
      : "memory");
}

// TMEM allocation for a CTA pair: executed by the same warp in both CTAs.
__device__ __forceinline__ void tmem_alloc_pair(uint32_t* smem_result, uint32_t cols) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(smem_result)),
               "r"(cols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc_pair(uint32_t taddr, uint32_t cols) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(cols) : "memory");
}
// Whole-warp call (pair leader): one elected lane issues the 4 SS MMAs of a
// 128-byte K atom with cta_group::2 (M = 256 across the pair).
template <bool kTF32>
__device__ __forceinline__ void mma_ss_atom_pair_elect(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                                       uint32_t idesc, uint32_t accumulate) {
#define MEC_PAIR_ATOM(KIND)                                                                             \
  asm volatile(                                                                                         \
      "{\n\t.reg .pred p, e;\n\t.reg .b64 a1, a2, a3, b1, b2, b3;\n\t"                                    \
      "setp.ne.b32 p, %4, 0;\n\t"                                                                       \
      "add.u64 a1, %1, 2;\n\tadd.u64 a2, %1, 4;\n\tadd.u64 a3, %1, 6;\n\t"                                 \
      "add.u64 b1, %2, 2;\n\tadd.u64 b2, %2, 4;\n\tadd.u64 b3, %2, 6;\n\t"                                 \
      "elect.sync _|e, 0xffffffff;\n\t"                                                                 \
      "@e tcgen05.mma.cta_group::2.kind::" KIND " [%0], %1, %2, %3, p;\n\t"                              \
      "@e tcgen05.mma.cta_group::2.kind::" KIND " [%0], a1, b1, %3, 1;\n\t"                              \
      "@e tcgen05.mma.cta_group::2.kind::" KIND " [%0], a2, b2, %3, 1;\n\t"                              \
      "@e tcgen05.mma.cta_group::2.kind::" KIND " [%0], a3, b3, %3, 1;\n\t}" ::"r"(tmem_d),              \
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)                                               \
      : "memory")
  if constexpr (kTF32) {
    MEC_PAIR_ATOM("tf32");
  } else {
    MEC_PAIR_ATOM("f16");
  }
#undef MEC_PAIR_ATOM
}
// As mma_ss_atom_pair_elect with B advanced by b_step (16-byte units) per
// 32-byte K step instead of 2 (an MN-major B: one K step = 16 bf16 / 8 tf32
// K rows = b_step x 16 bytes further on).
template <bool kTF32>
__device__ __forceinline__ void mma_ss_atom_pair_bstep_elect(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                                             uint32_t b_step, uint32_t idesc, uint32_t accumulate) {
#define MEC_PAIR_ATOM_BS(KIND)                                                                          \
  asm volatile(                                                                                         \
      "{\n\t.reg .pred p, e;\n\t.reg .b64 a1, a2, a3, b1, b2, b3, s;\n\t"                                 \
      "setp.ne.b32 p, %5, 0;\n\t"                                                                       \
      "cvt.u64.u32 s, %3;\n\t"                                                                           \
      "add.u64 a1, %1, 2;\n\tadd.u64 a2, %1, 4;\n\tadd.u64 a3, %1, 6;\n\t"                                 \
      "add.u64 b1, %2, s;\n\tadd.u64 b2, b1, s;\n\tadd.u64 b3, b2, s;\n\t"                               \
      "elect.sync _|e, 0xffffffff;\n\t"                                                                 \
      "@e tcgen05.mma.cta_group::2.kind::" KIND " [%0], %1, %2, %4, p;\n\t"                              \
      "@e tcgen05.mma.cta_group::2.kind::" KIND " [%0], a1, b1, %4, 1;\n\t"                              \
      "@e tcgen05.mma.cta_group::2.kind::" KIND " [%0], a2, b2, %4, 1;\n\t"                              \
      "@e tcgen05.mma.cta_group::2.kind::" KIND " [%0], a3, b3, %4, 1;\n\t}" ::"r"(tmem_d),              \
      "l"(adesc), "l"(bdesc), "r"(b_step), "r"(idesc), "r"(accumulate)                                  \
      : "memory")
  if constexpr (kTF32) {
    MEC_PAIR_ATOM_BS("tf32");
  } else {
    MEC_PAIR_ATOM_BS("f16");
  }
#undef MEC_PAIR_ATOM_BS
}

// Whole-warp call (pair leader): commit the pair's prior MMAs to the mbarrier
// at the same shared offset in every CTA of `cta_mask` (multicast arrive).
__device__ __forceinline__ void mma_commit_pair_elect(uint64_t* bar, uint16_t cta_mask) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}" ::"r"(
          smem_u32(bar)),
      "h"(cta_mask)
      : "memory");
}
// 16-byte global load that bypasses L1 (data written by other SMs in this launch)
__device__ __forceinline__ uint4 ld_global_cg_v4(const void* p) {
  uint4 v;
  asm volatile("ld.global.cg.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}

// ----------------------------------------------------------- descriptors
// Shared-memory matrix descriptor (tcgen05 "matrix descriptor"), K-major
// operand stored in the canonical 128-byte-swizzle layout that a TMA load with
// CU_TENSOR_MAP_SWIZZLE_128B and a 128-byte inner box produces: rows of 128 B,
// 8-row (1024 B) swizzle atoms.  Fields: start>>4 [0,14), LBO>>4 [16,30)
// (unused for swizzled K-major; 1), SBO>>4 [32,46) = 1024>>4, version [46,48)
// = 1, base offset [49,52) = 0, layout [61,64) = 2 (SWIZZLE_128B).
__device__ __forceinline__ uint64_t smem_desc_sw128(uint32_t smem_addr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((smem_addr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>(1) << 16;
  d |= static_cast<uint64_t>(1024 >> 4) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(2) << 61;
  return d;
}

// MN-major operand (N contiguous) in the 128-byte-swizzle canonical layout a
// TMA load of {128 bytes of N, K rows} boxes with CU_TENSOR_MAP_SWIZZLE_128B
// produces: 8 K-rows of 128 B form a 1 KB swizzle atom (SBO = 1024 B between
// consecutive groups of 8 K rows), and consecutive 128-byte N chunks are
// lbo_bytes apart (LBO: one box).
__device__ __forceinline__ uint64_t smem_desc_sw128_mn(uint32_t smem_addr, uint32_t lbo_bytes) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((smem_addr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= static_cast<uint64_t>(1024 >> 4) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(2) << 61;
  return d;
}

// Instruction descriptor (kind::f16 / kind::tf32): D fp32 [4,6)=1,
// A/B format [7,10)/[10,13) (1 = BF16, 2 = TF32), both K-major (bits 15,16 = 0),
// N>>3 at [17,23), M>>4 at [24,29).
__host__ __device__ constexpr uint32_t instr_desc(bool tf32, uint32_t M, uint32_t N, bool b_mn = false) {
  return (1u << 4) | ((tf32 ? 2u : 1u) << 7) | ((tf32 ? 2u : 1u) << 10) | ((b_mn ? 1u : 0u) << 16) |
         ((N >> 3) << 17) | ((M >> 4) << 24);
}

}  // namespace ptx
}  // namespace mec
