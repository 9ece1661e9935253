// tcgen05 (5th-generation tensor core) primitives for sm_100a, raw PTX:
// TMEM allocation, shared-memory matrix descriptors, the kind::f16 MMA,
// commit-to-mbarrier and TMEM -> register loads.
//
// Operand layout used throughout (no swizzle, "interleaved" core matrices):
// a bf16 matrix stored as [rows][cols] is blocked into 8 x 8 core matrices of
// 128 contiguous bytes (8 rows of 16 B); the core matrices of one 8-row group
// are contiguous along cols:
//     byte(r, c) = (r / 8) * (cols / 8) * 128 + (c / 8) * 128 + (r % 8) * 16 + (c % 8) * 2
// The SAME buffer is a K-major operand when cols is the MMA's K dimension
// (leading byte offset = 128, stride byte offset = cols / 8 * 128) and an
// MN-major operand when rows is K (the 16-byte rows of a core matrix then run
// along MN: stride byte offset = 128 between MN-adjacent core matrices,
// leading byte offset = cols / 8 * 128 between K-adjacent ones) -- so a tile of
// activations written once serves as the A operand of the next layer's GEMM
// and, transposed, as an operand of the weight-gradient GEMM.
#pragma once
#include <cuda_bf16.h>

#include "qs_common.cuh"

namespace umma {

// element offset (in bf16 elements) of (r, c) in the blocked layout
QS_D int blk_off(int r, int c, int cols) { return ((r >> 3) * (cols >> 3) + (c >> 3)) * 64 + (r & 7) * 8 + (c & 7); }

// shared-memory matrix descriptor (tcgen05 "matrix descriptor"): start address,
// leading / stride byte offsets (>> 4), version 1 (sm_100), no swizzle
QS_D uint64_t smem_desc(const void* p, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(p);
  uint64_t d = 0;
  d |= (uint64_t)((a >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;  // version
  // base offset 0, lbo mode 0, layout type 0 (SWIZZLE_NONE)
  return d;
}
// K-major view of a [rows=MN][cols=K] blocked buffer; MN-major view of a
// [rows=K][cols=MN] blocked buffer (see the header comment)
QS_D uint64_t desc_kmajor(const void* p, int cols) { return smem_desc(p, 128, (uint32_t)(cols >> 3) * 128); }
QS_D uint64_t desc_mnmajor(const void* p, int cols) { return smem_desc(p, (uint32_t)(cols >> 3) * 128, 128); }

// instruction descriptor, kind::f16: D fp32, A and B bf16, dense
QS_HD uint32_t idesc_bf16(int M, int N, bool a_mn_major, bool b_mn_major) {
  uint32_t d = 0;
  d |= 1u << 4;   // D format F32
  d |= 1u << 7;   // A format BF16
  d |= 1u << 10;  // B format BF16
  d |= (a_mn_major ? 1u : 0u) << 15;
  d |= (b_mn_major ? 1u : 0u) << 16;
  d |= (uint32_t)(N >> 3) << 17;
  d |= (uint32_t)(M >> 4) << 24;
  return d;
}

// D[tmem] (+)= A[smem] B[smem], issued by one thread
QS_D void mma_bf16(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc, bool accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
      ::"r"(d_tmem), "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate ? 1 : 0));
}

// arrive on an mbarrier once every previously issued tcgen05.mma of this thread completed
QS_D void commit(uint64_t* mbar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(mbar))
               : "memory");
}

QS_D void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
QS_D void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
// generic-proxy shared-memory writes -> visible to the tensor core's async proxy
QS_D void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// one warp: allocate / free `cols` TMEM columns (power of 2 >= 32)
QS_D void tmem_alloc(uint32_t* smem_result, uint32_t cols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(smem_result)),
               "r"(cols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
QS_D void tmem_free(uint32_t taddr, uint32_t cols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(cols) : "memory");
}

// 32 lanes x 16 columns of 32-bit: thread i of the warp gets lane (base lane + i),
// columns [col, col + 16)
QS_D void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// the same for 32 columns [col, col + 32): one load, one wait
QS_D void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// TMEM address of (lane, column)
QS_D uint32_t taddr(uint32_t base, int lane, int col) { return base + ((uint32_t)lane << 16) + (uint32_t)col; }

QS_D void mbar_wait_parity(uint64_t* bar, uint32_t parity) { mbar_wait(bar, parity); }

}  // namespace umma
