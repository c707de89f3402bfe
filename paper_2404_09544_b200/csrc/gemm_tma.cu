// Dense transform of the GNN layer on tcgen05 with TMA-fed fp32 operands
// (kind::tf32, fp32 accumulation in TMEM) -- the GNNV_PREC_TF32 path.
//
// Paper: Eq.1 Combine; Algorithm 1 lines 6 and 8.
//
// Why tf32 + TMA: at hidden 256 the layer GEMMs have low arithmetic
// intensity against fp32 activations (e.g. products layer 1: 50 GFLOP on
// 0.9 GB), so they are HBM-bound on B200 even at tf32 rates (~1.1 PF dense).
// Feeding the fp32 activations to the tensor cores as tf32 removes every
// conversion pass: TMA writes the tiles straight into the UMMA canonical
// 128B-swizzled layout and the MMA consumes them in place.
//
//   fwd : Y = act([X1 | X2] W + b)   A = activations, K-major (TMA box 128 x 32)
//                                     B = W^T, K-major (prep image [Npad x K'])
//   dX  : [Y1 | Y2] = G W^T           A = G, K-major; B = W rows, K-major image
//   dW  : dW = [X1 | X2]^T G'         operands arrive MN-major (TMA boxes of 16
//                                     graph rows x 128/256 columns, unswizzled);
//                                     kind::tf32 only takes K-major operands (an
//                                     MN-major tf32 operand yields zeros on
//                                     sm_100a), so the NE transposer warps turn
//                                     each staged box into double-buffered
//                                     K-major SW64 tiles (conflict-free rotated
//                                     STS.128) and, on the way, apply the ReLU
//                                     bits to G and sum db = colsum(G').  The
//                                     reduction over graph rows is split across
//                                     CTAs; split-K partials and db are added
//                                     into dW/db with red.global.add.f32
//                                     (arrival order, see include/gnnv.h).
//
// Warp roles (NTHREADS = 64 + 32*NE = 320): warp 0 = TMA producer (one
// elected thread), warp 1 = TMEM owner + MMA issuer (one elected thread),
// warps 2..2+NE-1 = epilogue (fwd/dX: tcgen05.ld of TMEM lanes
// 32*(warp%4) .. +31, two warps per lane quadrant splitting the columns;
// bias, ReLU, ReLU bits, TMA store through a 128B-swizzled smem buffer) or
// transposers (dW).  fwd/dX are persistent over output tiles with two TMEM
// accumulators (epilogue of tile t overlaps the mainloop of tile t+1); dW
// owns one (i-tile group, row split) per CTA.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cuda_bf16.h>

#include "common.cuh"

namespace gnnv {
namespace tma {

constexpr int BM = 128;     // MMA M
constexpr int BKB = 128;    // bytes of K per stage row (32 fp32 = one 128B swizzle atom row)
constexpr int BK = 32;      // fp32 elements of K per stage
constexpr int NE = 8;       // epilogue / transposer warps
constexpr int NTHREADS = 64 + 32 * NE;
constexpr int FWD_STAGES = 4;
constexpr int PAIR_STAGES = 5;  // CTA-pair fwd: a stage is A 16 KB + half of B 16 KB
constexpr int PAIR_OB = 2;      // CTA-pair fwd: double-buffered 4 KB epilogue staging per warp
constexpr int DW_STAGES = 4;
constexpr int DW_STAGES16 = 6;  // dW with a bf16 G: 24 KB stages, two more in flight
constexpr int DW_MT = 2;    // 128-row i-tiles per dW CTA
constexpr int DW_KR = 16;   // graph rows per dW k-block
constexpr int MODE_FWD = 0, MODE_DX = 1, MODE_DW = 2;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* b, uint32_t tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(tx) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 1000000;\n@!p bra W_%=;\n}\n" ::"r"(
          smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tc_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
// TMA gather4 (sm_100a): rows r0..r3 of a 2-D tensor, columns [c0, c0 + box
// width), into 4 consecutive box rows at dst (the tensor map's box is
// {width, 1}); the swizzle follows the shared-memory address as for tiles.
__device__ __forceinline__ void tma_gather4(void* dst, const CUtensorMap* map, int c0, int r0, int r1, int r2, int r3,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
      "%4, %5, %6}], [%7];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(map), "r"(c0),
               "r"(c1), "r"(smem_u32(src))
               : "memory");
}
__device__ __forceinline__ void st_shared_v4(uint32_t addr, float a, float b, float c, float d) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
}
__device__ __forceinline__ void tma_prefetch(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(map) : "memory");
}

// K-major swizzled descriptors (sm100 version 1).  SW128: rows of 128B
// (32 tf32 of K), 8-row atoms 1024B apart (SBO); SW64: rows of 64B, 8-row
// atoms of 512B.  The K step of 8 tf32 moves the start address by 32B.
__device__ __forceinline__ uint64_t desc_sw(uint32_t saddr, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1 << 16;  // LBO (unused for swizzled K-major)
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)layout << 61;  // 2 = SWIZZLE_128B, 4 = SWIZZLE_64B
  return d;
}
// kind::tf32 instruction descriptor: D=f32, A=B=tf32, M=128, N, majors.
__device__ __forceinline__ uint32_t idesc_tf32(uint32_t n, bool a_mn, bool b_mn, uint32_t m = BM) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((a_mn ? 1u : 0u) << 15) | ((b_mn ? 1u : 0u) << 16) | ((n >> 3) << 17) |
         ((m >> 4) << 24);
}
__device__ __forceinline__ void mma_tf32(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(
          d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
// ---- CTA pair (cluster of 2, tcgen05 cta_group::2) helpers
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cluster address of the same offset in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t map_rank(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1, 1000000;\n@!p bra "
      "W_%=;\n}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
// TMA into this CTA's shared memory, completing bytes on the pair leader's
// mbarrier (rank 0: the barrier address with the peer bit cleared)
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
      "[%4];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar) & 0xFEFFFFFFu)
      : "memory");
}
__device__ __forceinline__ void mma_tf32_pair(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
// arrive on the barrier at this offset in both CTAs of the pair when the
// leader's MMAs issued so far complete
__device__ __forceinline__ void mma_commit_pair(uint64_t* bar) {
  asm volatile(
      "{\n.reg .b16 m;\nmov.b16 m, 3;\ntcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 "
      "[%0], m;\n}\n" ::"r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mma_f16(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
// kind::f16 instruction descriptor: D=f32, A=B=bf16, M=128, N, majors.
__device__ __forceinline__ uint32_t idesc_bf16(uint32_t n, bool a_mn, bool b_mn, uint32_t m = BM) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((a_mn ? 1u : 0u) << 15) | ((b_mn ? 1u : 0u) << 16) | ((n >> 3) << 17) |
         ((m >> 4) << 24);
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr)
      : "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,"
      "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr)
      : "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// tcgen05.ld without the wait (several loads in flight; tmem_wait_ld32
// then waits and pins the registers after the wait)
__device__ __forceinline__ void tmem_ld32_nw(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,"
      "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr)
      : "memory");
}
__device__ __forceinline__ void tmem_ld16_nw(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr)
      : "memory");
#pragma unroll
  for (int i = 16; i < 32; ++i) r[i] = 0u;
}
__device__ __forceinline__ void tmem_pin32(uint32_t (&r)[32]) {
  asm volatile(""
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                 "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]), "+r"(r[15]),
                 "+r"(r[16]), "+r"(r[17]), "+r"(r[18]), "+r"(r[19]), "+r"(r[20]), "+r"(r[21]), "+r"(r[22]),
                 "+r"(r[23]), "+r"(r[24]), "+r"(r[25]), "+r"(r[26]), "+r"(r[27]), "+r"(r[28]), "+r"(r[29]),
                 "+r"(r[30]), "+r"(r[31]));
}

struct Params {
  CUtensorMap ta1, ta2, tb;
  CUtensorMap ty1, ty2;  // fwd/dX outputs (TMA stores, SW128 boxes of 32 x 32)
  CUtensorMap ty16;      // fwd: the bf16 copy (unswizzled boxes of 32 x 32 bf16)
  int two;      // A has a second source (SAGE [H_dst | A])
  int f16;      // fwd: bf16 operands (kind::f16; 64-element k-blocks, same 128-byte rows)
  int bres;     // fwd: B (W^T) loaded once per CTA and kept resident; stages carry A only
  int eppipe;   // fwd bf16 epilogue: next pass's TMEM loads issued before this pass's fence
  int nkb1;     // fwd: K blocks served by X1 (ceil(K1/32)); dw: 32-col blocks of X1
  int nkb;      // fwd/dx: K blocks in total
  int BN;       // N per tile (fwd/dx: mult of 16; dw: mult of 32)
  int n_ntiles; // dx
  const int32_t* dM;
  // fwd epilogue
  float* Y;
  int ldy, N;
  const float* bias;
  int relu;
  // dx epilogue
  float *Y1, *Y2;
  int ld1, ld2;
  // dw: outputs accumulated atomically (zeroed by the host side first)
  float* dW;
  float* db;
  int K1;
  int splits, ablocks;  // ablocks: valid 32-wide i blocks (X1 then X2)
  // dw with a fused ReLU mask: G' = G * bit and db partials per split; th =
  // the [M x nwp] uint32 bit mask (TMA box DW_KR x nwp)
  CUtensorMap th;
  int mask, nwp;
  // fwd with relu: bit mask output (NULL: none)
  uint32_t* bits;
  int bits_ld;
  // dX: multiply the Y1 columns by a ReLU bit mask (the previous layer's),
  // ybits[m*ybits_ld + col/32] (NULL: none)
  const uint32_t* ybits;
  int ybits_ld;
  // dW: also the column sums of G (db) without a mask (G already masked)
  int dbsum;
  // fwd / dW: X1 row m is row x1_rows[m] of the tensor behind ta1 (layer 1
  // reading H_dst straight from the degree-ordered cache table): ta1 then
  // has a {width, 1} box and X1 tiles arrive by TMA gather4, 4 rows per
  // instruction, one instruction per producer lane (NULL: plain tiles)
  const int32_t* x1_rows;
  // fwd: the next layer's aggregation fused into this epilogue (see
  // GemmFwdArgs::push_*); push_out NULL = off
  const int32_t* push_colptr;
  const int32_t* push_dst;
  const int32_t* push_indptr;
  float* push_out;
  int push_ld, push_mean;
  const int32_t* keep_rows;
  const int32_t* push_owner;  // owner row of each output row (-1: none); its edge is not in the CSC
  // bf16 copies (the trainer's bf16 intermediates):
  // fwd: every output row also stored as bf16 (y16, stride ld16, a multiple
  // of 32), the fp32 rows only below *keep_rows; dX: the Y1 part stored as
  // bf16 (y1_16, stride ld1) instead of fp32; dW: G is bf16 (g16 = 1)
  __nv_bfloat16* y16;
  int ld16;
  __nv_bfloat16* y1_16;
  __nv_bfloat16* y2_16;  // dX: Y2 (dA) as bf16 too
  CUtensorMap ty2_16;
  int g16;
  // fwd/dX (not PAIR): dynamic tile scheduler -- [0] next tile counter,
  // [1] finished CTAs (the last one resets both); NULL: static round robin
  unsigned int* sched;
};


__device__ __forceinline__ uint32_t bf16x2(float a, float b) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<const uint32_t*>(&h);
}

// The last CTA of a launch to finish resets its scheduler slot for the next
// launch that draws it (all producers' claims precede every CTA's exit).
__device__ __forceinline__ void sched_done(unsigned int* sched) {
  __threadfence();
  if (atomicAdd(sched + 1, 1u) == gridDim.x * gridDim.y - 1) {
    sched[0] = 0u;
    sched[1] = 0u;
    __threadfence();
  }
}
__device__ unsigned int g_sched[4096][2];  // zero-initialised; a ring of slots, one per launch in flight (a slot is reused only 4096 launches later -- beyond any launch queue)

// PAIR (MODE_FWD only): a cluster of 2 CTAs computes 256-row tiles with
// tcgen05.mma.cta_group::2 (M = 256): each CTA stages its own 128 rows of A
// and half of the W^T tile's N columns, the leader (rank 0) issues the MMAs,
// each CTA's TMEM receives its 128 rows; the W^T bytes each CTA pulls from L2
// per k-block halve, and the smaller stage affords 6 stages.
template <int MODE, bool PAIR = false>
__global__ void __launch_bounds__(NTHREADS, 1) k_tma_gemm(const __grid_constant__ Params p) {
  GNNV_PDL_ENTRY();
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ __align__(16) float s_bias[256];
  // dynamic tile scheduler (fwd/dX, not PAIR): the producer claims tiles
  // (its CTA's first tile statically, then atomically from p.sched) and
  // publishes each in a ring slot; the MMA and epilogue warps take them in
  // the same order.  A CTA that starts late -- its SM still held by the
  // concurrent Eq.4 prefetch -- then simply processes fewer tiles.  The
  // producer runs at most FWD_STAGES k-blocks ahead of the MMA, which runs at
  // most two tiles ahead of the epilogue, so 8 slots are never overrun.

  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  const int S = MODE == MODE_DW ? (p.g16 ? DW_STAGES16 : DW_STAGES) : PAIR ? PAIR_STAGES : FWD_STAGES;
  constexpr int MT = MODE == MODE_DW ? DW_MT : 1;
  const int BN = p.BN;
  const uint32_t crank = PAIR ? cluster_rank() : 0u;
  const int pid = PAIR ? (int)blockIdx.x / 2 : (int)blockIdx.x;   // tile-loop index of this CTA (pair)
  const int npid = PAIR ? (int)gridDim.x / 2 : (int)gridDim.x;
  // fwd/dX stage: A [128 rows x 128B] + B [BN rows x 128B] (K-major SW128 boxes;
  // PAIR: B [BN/2 rows x 128B], this CTA's half of N).
  // dW stage (unswizzled row-major boxes of DW_KR graph rows): MT A tiles of
  // [16 x 128] fp32, then G [16 x BN], then (fused mask) H [16 x BN].
  const int a_bytes = MODE == MODE_DW ? MT * DW_KR * BM * 4 : BM * BKB;
  const int g_bytes = MODE == MODE_DW ? DW_KR * BN * (p.g16 ? 2 : 4) : (PAIR ? BN / 2 : BN) * BKB;
  const bool bres = MODE == MODE_FWD && !PAIR && p.bres;
  const int b_bytes = MODE == MODE_DW ? g_bytes + (p.mask ? DW_KR * p.nwp * 4 : 0) : bres ? 0 : g_bytes;
  const int stage_bytes = a_bytes + b_bytes;
  // resident B (bres): the nkb k-blocks of W^T [BN rows x 128B] first, then the A stages
  uint8_t* sres = smem;
  uint8_t* sst = smem + (bres ? (size_t)p.nkb * g_bytes : (size_t)0);
  // dW: two K-major SW64 tiles (64B rows = 16 tf32 of K) built by the transposers;
  // fwd/dX: one 4 KB SW128 output staging buffer per epilogue warp (TMA store)
  const int kt_bytes = MODE == MODE_DW ? (MT * BM + BN) * 64 : 0;
  uint8_t* kbuf = sst + (((size_t)S * stage_bytes + 1023) & ~(size_t)1023);  // swizzle-atom aligned
  uint8_t* obuf = kbuf;
  const int extra = MODE == MODE_DW ? 2 * kt_bytes : NE * 4096 * (PAIR ? PAIR_OB : 1);
  uint64_t* bars = reinterpret_cast<uint64_t*>(kbuf + extra);
  uint64_t* full = bars;
  uint64_t* empty = bars + S;
  uint64_t* kready = bars + 2 * S;  // dW: K-major tile b ready
  uint64_t* kfree = kready + 2;     // dW: MMA finished reading tile b
  uint64_t* tfull = kfree + 2;      // fwd/dX: two TMEM accumulators
  uint64_t* tempty = tfull + 2;
  uint64_t* s_tbar = tempty + 2;                          // [8] tile ring barriers
  int* s_tile = reinterpret_cast<int*>(s_tbar + 8);       // [8] tile ring slots
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(s_tile + 8);
  uint64_t* bfull = reinterpret_cast<uint64_t*>(s_tmem + 2);  // bres: W^T resident
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int M = *p.dM;

  int ntiles = 0, kb0 = 0, kb1 = 0;
  if (MODE == MODE_DW) {
    const int nkbm = (M + DW_KR - 1) / DW_KR;
    const int per = (nkbm + p.splits - 1) / p.splits;
    kb0 = min(nkbm, (int)blockIdx.x * per);
    kb1 = min(nkbm, kb0 + per);
  } else {
    ntiles = ((M + BM - 1) / BM) * (MODE == MODE_DX ? p.n_ntiles : 1);
    if (PAIR) ntiles = (ntiles + 1) / 2;  // 256-row pair tiles
    if (pid >= ntiles) {  // block-uniform (pair-uniform)
      if (!PAIR && p.sched && threadIdx.x == 0) sched_done(p.sched);
      return;
    }
  }
  const bool dyn = MODE != MODE_DW && !PAIR && p.sched != nullptr;
  uint32_t ncols = 32;
  const uint32_t need = (uint32_t)(MT * BN) * (MODE == MODE_DW ? 1u : 2u);
  while (ncols < need) ncols <<= 1;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], MODE == MODE_DW ? NE : 1);  // dW: released by the transposer warps (one arrive each)
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&kready[b], NE);
      mbar_init(&kfree[b], 1);
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], PAIR ? 2 * NE : NE);  // PAIR: the leader's, both CTAs' epilogue warps
    }
    for (int i = 0; i < 8; ++i) mbar_init(&s_tbar[i], 1);
    mbar_init(bfull, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (PAIR) cluster_sync_all();  // the peer's barriers exist before any remote arrive / TMA
  if (warp == 0 && lane == 0) {
    tma_prefetch(&p.ta1);
    if (p.two) tma_prefetch(&p.ta2);
    tma_prefetch(&p.tb);
  }
  if (warp == 1) {
    if (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(s_tmem)),
                   "r"(ncols)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(s_tmem)),
                   "r"(ncols)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
  }
  if (MODE == MODE_FWD && warp >= 2) {
    for (int i = threadIdx.x - 64; i < BN; i += NE * 32) s_bias[i] = i < p.N ? __ldg(p.bias + i) : 0.f;
  }
  tc_before();
  __syncthreads();
  tc_after();
  const uint32_t tmem = *s_tmem;

  if (MODE != MODE_DW) {
    // ======================= persistent fwd / dX =======================
    if (warp == 0) {
      const bool g4 = MODE == MODE_FWD && !PAIR && p.x1_rows != nullptr;
      if (PAIR) {
        if (lane == 0) {
          // both CTAs: wait for the local stage to be free (the leader's MMA
          // commit arrives on it in both CTAs), load this CTA's A rows and
          // half of B, completing bytes on the leader's full barrier
          int it = 0;
          for (int tile = pid; tile < ntiles; tile += npid) {
            const int mt = 2 * tile + (int)crank;
            for (int kb = 0; kb < p.nkb; ++kb, ++it) {
              const int s = it % S;
              uint8_t* sa = smem + (size_t)s * stage_bytes;
              uint8_t* sb = sa + a_bytes;
              if (it >= S) mbar_wait(&empty[s], ((it / S) & 1) ^ 1);
              if (crank == 0) mbar_arrive_tx(&full[s], (uint32_t)(2 * stage_bytes));
              if (kb >= p.nkb1) tma_load_2d_pair(sa, &p.ta2, (kb - p.nkb1) * BK, mt * BM, &full[s]);
              else tma_load_2d_pair(sa, &p.ta1, kb * BK, mt * BM, &full[s]);
              tma_load_2d_pair(sb, &p.tb, kb * BK, (int)crank * (BN / 2), &full[s]);
            }
          }
        }
      } else if (lane == 0 || g4) {
        int it = 0, lt = 0;
        for (int tile = blockIdx.x;; ++lt) {
          if (dyn && lane == 0) {  // publish the tile (or the end) to the MMA and epilogue warps
            s_tile[lt & 7] = tile < ntiles ? tile : -1;
            mbar_arrive(&s_tbar[lt & 7]);
          }
          if (tile >= ntiles) break;
          const int mt = MODE == MODE_DX ? tile / p.n_ntiles : tile;
          const int nt = MODE == MODE_DX ? tile % p.n_ntiles : 0;
          // gather4: lane l loads rows 4l..4l+3 of the tile; rows >= M read
          // table row 0 (their outputs are never stored)
          int r4[4] = {0, 0, 0, 0};
          if (g4) {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const int m = mt * BM + 4 * lane + j;
              r4[j] = m < M ? __ldg(p.x1_rows + m) : 0;
            }
          }
          if (bres && lt == 0 && lane == 0) {  // W^T once: nkb boxes on their own barrier
            mbar_arrive_tx(bfull, (uint32_t)(p.nkb * g_bytes));
            for (int kb = 0; kb < p.nkb; ++kb)
              tma_load_2d(sres + (size_t)kb * g_bytes, &p.tb, kb * (p.f16 ? 2 * BK : BK), 0, bfull);
          }
          for (int kb = 0; kb < p.nkb; ++kb, ++it) {
            const int s = it % S;
            uint8_t* sa = sst + (size_t)s * stage_bytes;
            uint8_t* sb = sa + a_bytes;
            if (lane == 0) {
              if (it >= S) mbar_wait(&empty[s], ((it / S) & 1) ^ 1);
              mbar_arrive_tx(&full[s], (uint32_t)stage_bytes);
            }
            if (g4) __syncwarp();
            const int kc = p.f16 ? 2 * BK : BK;  // elements per 128-byte k-block
            if (MODE == MODE_FWD && kb >= p.nkb1) {
              if (lane == 0) tma_load_2d(sa, &p.ta2, (kb - p.nkb1) * kc, mt * BM, &full[s]);
            } else if (g4) {
              tma_gather4(sa + lane * 4 * BKB, &p.ta1, kb * BK, r4[0], r4[1], r4[2], r4[3], &full[s]);
            } else {
              tma_load_2d(sa, &p.ta1, kb * kc, mt * BM, &full[s]);
            }
            if (lane == 0 && !bres) tma_load_2d(sb, &p.tb, kb * kc, nt * BN, &full[s]);
          }
          if (dyn) {
            int next = 0;
            if (lane == 0) next = (int)gridDim.x + (int)atomicAdd(p.sched, 1u);
            tile = g4 ? __shfl_sync(0xffffffffu, next, 0) : next;
          } else {
            tile += gridDim.x;
          }
        }
      }
    } else if (warp == 1) {
      if (PAIR) {
        if (lane == 0 && crank == 0) {
          const uint32_t idesc = idesc_tf32((uint32_t)BN, false, false, 2 * BM);
          int it = 0, lt = 0;
          for (int tile = pid; tile < ntiles; tile += npid, ++lt) {
            const int acc = lt & 1;
            if (lt >= 2) mbar_wait_cluster(&tempty[acc], ((lt >> 1) & 1) ^ 1);
            tc_after();
            for (int kb = 0; kb < p.nkb; ++kb, ++it) {
              const int s = it % S;
              mbar_wait(&full[s], (it / S) & 1);
              tc_after();
              const uint32_t a0 = smem_u32(smem + (size_t)s * stage_bytes);
              const uint32_t b0 = a0 + a_bytes;
#pragma unroll
              for (int k = 0; k < BK / 8; ++k)
                mma_tf32_pair(tmem + (uint32_t)(acc * BN), desc_sw(a0 + k * 32, 1024, 2),
                              desc_sw(b0 + k * 32, 1024, 2), idesc, (kb > 0 || k > 0) ? 1u : 0u);
              mma_commit_pair(&empty[s]);
            }
            mma_commit_pair(&tfull[acc]);
          }
        }
        __syncwarp();
      } else if (lane == 0) {
        const bool f16 = p.f16 != 0;
        const uint32_t idesc = f16 ? idesc_bf16((uint32_t)BN, false, false) : idesc_tf32((uint32_t)BN, false, false);
        int it = 0, lt = 0;
        for (int tile = blockIdx.x;; tile += gridDim.x, ++lt) {
          if (dyn) {
            mbar_wait(&s_tbar[lt & 7], (lt >> 3) & 1);
            tile = s_tile[lt & 7];
            if (tile < 0) break;
          } else if (tile >= ntiles) {
            break;
          }
          const int acc = lt & 1;
          if (lt >= 2) mbar_wait(&tempty[acc], ((lt >> 1) & 1) ^ 1);
          if (bres && lt == 0) mbar_wait(bfull, 0);
          tc_after();
          for (int kb = 0; kb < p.nkb; ++kb, ++it) {
            const int s = it % S;
            mbar_wait(&full[s], (it / S) & 1);
            tc_after();
            const uint32_t a0 = smem_u32(sst + (size_t)s * stage_bytes);
            const uint32_t b0 = bres ? smem_u32(sres + (size_t)kb * g_bytes) : a0 + a_bytes;
            // 32 bytes of K per MMA in both kinds (8 tf32 / 16 bf16)
            if (f16) {
#pragma unroll
              for (int k = 0; k < BK / 8; ++k)
                mma_f16(tmem + (uint32_t)(acc * BN), desc_sw(a0 + k * 32, 1024, 2), desc_sw(b0 + k * 32, 1024, 2),
                        idesc, (kb > 0 || k > 0) ? 1u : 0u);
            } else {
#pragma unroll
              for (int k = 0; k < BK / 8; ++k)
                mma_tf32(tmem + (uint32_t)(acc * BN), desc_sw(a0 + k * 32, 1024, 2), desc_sw(b0 + k * 32, 1024, 2),
                         idesc, (kb > 0 || k > 0) ? 1u : 0u);
            }
            mma_commit(&empty[s]);
          }
          mma_commit(&tfull[acc]);
        }
      }
      __syncwarp();
    } else {
      // 8 epilogue warps: TMEM lane quarter q = warp & 3 (tcgen05.ld
      // restriction), 32-column chunks interleaved between the two warps of a
      // quarter.  Each chunk (32 rows x 32 cols) goes through a 128B-swizzled
      // 4 KB smem buffer and one TMA store: coalesced full-line writes.
      const int q = warp & 3;
      const int half = (warp - 2) >> 2;
      constexpr int OBN = PAIR ? PAIR_OB : 1;
      uint8_t* ob0 = obuf + (warp - 2) * 4096 * OBN;
      int obi = 0;
      int y16h = 0;  // dX: the staging half of the next bf16 Y1 piece
      bool full_pending = false;  // the last TMA store read the whole 4 KB buffer
      int lt = 0;
      for (int tile = pid;; tile += npid, ++lt) {
        if (dyn) {
          mbar_wait(&s_tbar[lt & 7], (lt >> 3) & 1);
          tile = s_tile[lt & 7];
          if (tile < 0) break;
        } else if (tile >= ntiles) {
          break;
        }
        const int acc = lt & 1;
        const int mt = PAIR ? 2 * tile + (int)crank : MODE == MODE_DX ? tile / p.n_ntiles : tile;
        const int nt = MODE == MODE_DX ? tile % p.n_ntiles : 0;
        if (PAIR) mbar_wait_cluster(&tfull[acc], (lt >> 1) & 1);
        else mbar_wait(&tfull[acc], (lt >> 1) & 1);
        tc_after();
        const int row0 = mt * BM + q * 32;
        const uint32_t tbase = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN);
        // fused push of the next layer's aggregation: this warp's 32 rows'
        // in-edges (lane l: row row0 + l), an exclusive scan over the warp,
        // and the first 128 edges' (dst row, weight) held in registers
        // (edge p at lane p % 32, slot p / 32)
        const bool push = MODE == MODE_FWD && !PAIR && p.push_out != nullptr;
        int pe_beg = 0, pe_cnt = 0, pe_excl = 0, pe_incl = 0, pe_total = 0;
        int pv[4] = {0, 0, 0, 0};
        float pw[4] = {0.f, 0.f, 0.f, 0.f};
        bool store_rows = !(MODE == MODE_FWD && p.keep_rows) || row0 < *p.keep_rows;
        if (push) {
          const int u = row0 + lane;
          if (u < M) {
            pe_beg = __ldg(p.push_colptr + u);
            pe_cnt = __ldg(p.push_colptr + u + 1) - pe_beg;
          }
          pe_incl = pe_cnt;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, pe_incl, o);
            if (lane >= o) pe_incl += t;
          }
          pe_excl = pe_incl - pe_cnt;
          pe_total = __shfl_sync(0xffffffffu, pe_incl, 31);
          // edge pidx -> (row r, edge e): r = first lane whose inclusive
          // count exceeds pidx
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int pidx = k * 32 + lane;
            int r = 0;
            for (int b = 16; b; b >>= 1) {  // binary search over the warp's prefix counts
              const int cand = r + b;
              const int ci = __shfl_sync(0xffffffffu, pe_incl, cand - 1);
              if (ci <= pidx) r = cand;
            }
            const int eb = __shfl_sync(0xffffffffu, pe_beg, r), ex = __shfl_sync(0xffffffffu, pe_excl, r);
            if (pidx < pe_total) {
              const int v = __ldg(p.push_dst + eb + (pidx - ex));
              pv[k] = v | (r << 26);  // row index packed above the dst row (rows < 2^26)
              float w = 1.f;
              if (p.push_mean) {
                const int cv = __ldg(p.push_indptr + v + 1) - __ldg(p.push_indptr + v);
                w = cv ? 1.f / (float)cv : 0.f;
              }
              pw[k] = w;
            }
          }
        }
        // owner edges: row u's owner dst row (consecutive rows share it -- the
        // ids a dst row discovered are numbered consecutively by the relabel
        // scan), reduced as runs below; po_w = its mean weight
        int po = -1;
        float po_w = 0.f;
        if (push && p.push_owner) {
          const int u = row0 + lane;
          po = u < M ? __ldg(p.push_owner + u) : -1;
          if (po >= 0) {
            po_w = 1.f;
            if (p.push_mean) {
              const int cv = __ldg(p.push_indptr + po + 1) - __ldg(p.push_indptr + po);
              po_w = cv ? 1.f / (float)cv : 0.f;
            }
          }
        }
        if (MODE == MODE_FWD && !PAIR && p.y16 && !push) {
          // forward with the bf16 copy: two 32-column pieces per pass (64
          // contiguous columns; both TMEM loads in flight, one staging
          // round and one proxy fence for both bf16 pieces)
          const uint32_t ob_u32 = smem_u32(ob0);
          uint32_t r[2][32];
          // the next pass's TMEM loads are issued as soon as this pass's
          // packed pieces are in shared memory, so their latency overlaps
          // the proxy fence, the TMA stores and the ReLU-bit stores
          auto ld_pass = [&](int cp) {
#pragma unroll
            for (int h2 = 0; h2 < 2; ++h2) {
              const int c = cp + 32 * h2;
              if (c >= BN) continue;
              if (BN - c >= 32) tmem_ld32_nw(tbase + c, r[h2]);
              else tmem_ld16_nw(tbase + c, r[h2]);
            }
          };
          const bool epp = p.eppipe != 0;
          if (half * 64 < BN) ld_pass(half * 64);
          for (int c0 = half * 64; c0 < BN; c0 += 128) {
            if (!epp && c0 != half * 64) ld_pass(c0);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            tmem_pin32(r[0]);
            tmem_pin32(r[1]);
            const int64_t m = (int64_t)row0 + lane;
            const bool rag = row0 + 32 > M;
            uint32_t bw[2] = {0u, 0u};  // the pieces' ReLU bits, stored after the proxy fence
#pragma unroll
            for (int h2 = 0; h2 < 2; ++h2) {
              const int c = c0 + 32 * h2;
              if (c >= BN) continue;
              float v[32];
              uint32_t bits = 0;
              if (c + 32 <= p.N && p.relu) {  // whole piece inside N: vector bias loads, no column tests
                const float4* b4 = reinterpret_cast<const float4*>(s_bias + c);
#pragma unroll
                for (int j4 = 0; j4 < 8; ++j4) {
                  const float4 b = b4[j4];
                  v[4 * j4 + 0] = fmaxf(__uint_as_float(r[h2][4 * j4 + 0]) + b.x, 0.f);
                  v[4 * j4 + 1] = fmaxf(__uint_as_float(r[h2][4 * j4 + 1]) + b.y, 0.f);
                  v[4 * j4 + 2] = fmaxf(__uint_as_float(r[h2][4 * j4 + 2]) + b.z, 0.f);
                  v[4 * j4 + 3] = fmaxf(__uint_as_float(r[h2][4 * j4 + 3]) + b.w, 0.f);
                }
#pragma unroll
                for (int j = 0; j < 32; ++j) bits |= (v[j] > 0.f ? 1u : 0u) << j;
              } else {
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                  const int n = c + j;
                  float x = __uint_as_float(r[h2][j]) + (n < BN ? s_bias[n] : 0.f);
                  if (p.relu) x = fmaxf(x, 0.f);
                  v[j] = n < p.N ? x : 0.f;
                  bits |= (v[j] > 0.f ? 1u : 0u) << j;
                }
              }
              bw[h2] = bits;
              if (store_rows && rag) {  // ragged fp32 prefix rows: plain stores of the rows < M
                if (m < M)
#pragma unroll
                  for (int j = 0; j < 32; j += 4)
                    if (c + j < p.ldy)
                      *reinterpret_cast<float4*>(p.Y + m * p.ldy + c + j) =
                          make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
              } else if (store_rows) {  // fp32 prefix rows: 4 KB through the staging buffer
                if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                __syncwarp();
#pragma unroll
                for (int j = 0; j < 8; ++j)
                  st_shared_v4(ob_u32 + lane * 128 + ((j ^ (lane & 7)) << 4), v[4 * j], v[4 * j + 1], v[4 * j + 2],
                               v[4 * j + 3]);
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if (lane == 0) {
                  tma_store_2d(&p.ty1, ob0, c, row0);
                  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                }
              }
              // the bf16 piece: packed into r[h2][0..15] until both are staged
#pragma unroll
              for (int q = 0; q < 16; ++q) r[h2][q] = bf16x2(v[2 * q], v[2 * q + 1]);
            }
            if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            __syncwarp();
#pragma unroll
            for (int h2 = 0; h2 < 2; ++h2)
#pragma unroll
              for (int q = 0; q < 4; ++q)
                asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(ob_u32 + h2 * 2048 + lane * 64 + q * 16),
                             "r"(r[h2][4 * q]), "r"(r[h2][4 * q + 1]), "r"(r[h2][4 * q + 2]), "r"(r[h2][4 * q + 3])
                             : "memory");
            if (epp && c0 + 128 < BN) ld_pass(c0 + 128);
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) {
              for (int h2 = 0; h2 < 2; ++h2)
                if (c0 + 32 * h2 < BN && c0 + 32 * h2 < p.ld16) tma_store_2d(&p.ty16, ob0 + h2 * 2048, c0 + 32 * h2, row0);
              asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
            // the ReLU bits after the fence: a global store ahead of it would
            // hold the fence's CTA-scope membar for the store's round trip
            if (p.bits && m < M) {
              uint32_t* bp = p.bits + m * p.bits_ld + (c0 >> 5);
              bp[0] = bw[0];
              if (c0 + 32 < BN) bp[1] = bw[1];
            }
          }
        } else
        for (int c = half * 32; c < BN; c += 64) {
          float v[32];
          if (BN - c >= 32) tmem_ld32(tbase + c, v);
          else {
            tmem_ld16(tbase + c, v);
#pragma unroll
            for (int j = 16; j < 32; ++j) v[j] = 0.f;
          }
          if (MODE == MODE_FWD) {
            uint32_t bits = 0;
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const int n = c + j;
              float x = v[j] + (n < BN ? s_bias[n] : 0.f);
              if (p.relu) x = fmaxf(x, 0.f);
              v[j] = n < p.N ? x : 0.f;
              bits |= (v[j] > 0.f ? 1u : 0u) << j;
            }
            if (p.bits && row0 + lane < M) p.bits[(int64_t)(row0 + lane) * p.bits_ld + (c >> 5)] = bits;
          }
          const int j0 = nt * BN + c;  // dX: column in the [Y1 | Y2] space
          if (MODE == MODE_DX && p.ybits && j0 < p.ld1) {
            // G_src = (G W_s^T) * relu'(H_src): chunks are 32-aligned, one word
            const int64_t m = (int64_t)row0 + lane;
            const uint32_t wv = m < M ? __ldg(p.ybits + m * p.ybits_ld + (j0 >> 5)) : 0u;
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (j0 + j < p.ld1 && !((wv >> j) & 1u)) v[j] = 0.f;
          }
          // dX pieces stored as bf16: Y1 (dH_dst) and/or Y2 (dA)
          const bool y16c = MODE == MODE_DX && ((p.y1_16 && j0 < p.ld1) ||
                                                (p.y2_16 && j0 >= p.ld1 && j0 - p.ld1 + 32 <= p.ld2));
          if (y16c && row0 + 32 <= M) {
            // Y1 as bf16 (j0 + 32 <= ld1: checked on the host): the 2 KB
            // piece through a staging half and a TMA store (halves alternate,
            // so one store may still be reading while the next is written)
            const uint32_t hb = smem_u32(ob0) + (uint32_t)y16h * 2048u;
            if (lane == 0) {  // a 4 KB fp32 store issued last reads both halves
              if (full_pending) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
              else asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
            }
            full_pending = false;
            __syncwarp();
#pragma unroll
            for (int q = 0; q < 4; ++q)
              asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(hb + lane * 64 + q * 16),
                           "r"(bf16x2(v[8 * q], v[8 * q + 1])), "r"(bf16x2(v[8 * q + 2], v[8 * q + 3])),
                           "r"(bf16x2(v[8 * q + 4], v[8 * q + 5])), "r"(bf16x2(v[8 * q + 6], v[8 * q + 7]))
                           : "memory");
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) {
              if (j0 < p.ld1) tma_store_2d(&p.ty16, ob0 + y16h * 2048, j0, row0);
              else tma_store_2d(&p.ty2_16, ob0 + y16h * 2048, j0 - p.ld1, row0);
              asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
            y16h ^= 1;
            continue;
          }
          if (y16c) {  // ragged tile: the rows < M with plain stores
            const int64_t m = (int64_t)row0 + lane;
            if (m < M) {
              uint4* dst = j0 < p.ld1 ? reinterpret_cast<uint4*>(p.y1_16 + m * p.ld1 + j0)
                                      : reinterpret_cast<uint4*>(p.y2_16 + m * p.ld2 + (j0 - p.ld1));
#pragma unroll
              for (int q = 0; q < 4; ++q)
                dst[q] = make_uint4(bf16x2(v[8 * q], v[8 * q + 1]), bf16x2(v[8 * q + 2], v[8 * q + 3]),
                                    bf16x2(v[8 * q + 4], v[8 * q + 5]), bf16x2(v[8 * q + 6], v[8 * q + 7]));
            }
            continue;
          }
          const bool ragged = row0 + 32 > M || (MODE == MODE_DX && j0 < p.ld1 && j0 + 32 > p.ld1);
          if (ragged && store_rows) {
            // ragged last chunk: plain stores of the rows < M only (the TMA
            // map spans the row capacity, which may exceed the caller's rows);
            // a dX chunk straddling Y1 | Y2 also takes this path
            const int64_t m = (int64_t)row0 + lane;
            if (m < M) {
#pragma unroll
              for (int j = 0; j < 32; j += 4) {
                const float4 o = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
                if (MODE == MODE_FWD) {
                  if (c + j < p.ldy) *reinterpret_cast<float4*>(p.Y + m * p.ldy + c + j) = o;
                } else {
                  const int col = nt * BN + c + j;
                  if (col < p.ld1) *reinterpret_cast<float4*>(p.Y1 + m * p.ld1 + col) = o;
                  else if (p.Y2 && col - p.ld1 < p.ld2) *reinterpret_cast<float4*>(p.Y2 + m * p.ld2 + (col - p.ld1)) = o;
                }
              }
            }
          }
          if (MODE == MODE_FWD && !PAIR && p.y16 && !push) {
            // the bf16 copy (every row) -- and the fp32 dst-prefix rows
            // first, if this chunk has any -- through the staging buffer and
            // TMA stores.  The 2 KB bf16 pieces (32 rows x 64 bytes) alternate
            // between the buffer's halves, so one may still be read while
            // the next is written; the 4 KB fp32 piece waits for both
            uint8_t* ob = ob0;
            const uint32_t ob_u32 = smem_u32(ob);
            if (store_rows && !ragged) {
              if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
              __syncwarp();
#pragma unroll
              for (int j = 0; j < 8; ++j)
                st_shared_v4(ob_u32 + lane * 128 + ((j ^ (lane & 7)) << 4), v[4 * j], v[4 * j + 1], v[4 * j + 2],
                             v[4 * j + 3]);
              asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
              __syncwarp();
              if (lane == 0) {
                tma_store_2d(&p.ty1, ob, c, row0);
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
              }
              __syncwarp();
            }
            if (c < p.ld16) {
              const uint32_t hb = ob_u32 + (uint32_t)obi * 2048u;
              if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
              __syncwarp();
#pragma unroll
              for (int q = 0; q < 4; ++q)
                asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(hb + lane * 64 + q * 16),
                             "r"(bf16x2(v[8 * q], v[8 * q + 1])), "r"(bf16x2(v[8 * q + 2], v[8 * q + 3])),
                             "r"(bf16x2(v[8 * q + 4], v[8 * q + 5])), "r"(bf16x2(v[8 * q + 6], v[8 * q + 7]))
                             : "memory");
              asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
              __syncwarp();
              if (lane == 0) {
                tma_store_2d(&p.ty16, ob + obi * 2048, c, row0);
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
              }
              obi ^= 1;
            }
            continue;
          }
          if (ragged && !push) continue;
          if (!push && !store_rows) continue;
          // the TMA store that last used this buffer (OBN chunks ago) must
          // have read it; the OBN - 1 most recent ones may still be reading
          uint8_t* ob = ob0 + obi * 4096;
          const uint32_t ob_u32 = smem_u32(ob);
          obi = (obi + 1) % OBN;
          if (lane == 0) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(OBN - 1) : "memory");
          __syncwarp();
#pragma unroll
          for (int j = 0; j < 8; ++j)
            st_shared_v4(ob_u32 + lane * 128 + ((j ^ (lane & 7)) << 4), v[4 * j], v[4 * j + 1], v[4 * j + 2],
                         v[4 * j + 3]);
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0 && !ragged && store_rows) {
            if (MODE == MODE_FWD) {
              tma_store_2d(&p.ty1, ob, c, row0);
            } else if (j0 < p.ld1) {
              tma_store_2d(&p.ty1, ob, j0, row0);
            } else if (p.Y2) {
              tma_store_2d(&p.ty2, ob, j0 - p.ld1, row0);
            }
            full_pending = true;
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          }
          if (push && p.push_owner) {
            // owner edges as runs: lane j sums column c + j over the rows of
            // each run of equal owner rows (conflict-free LDS: one 128-byte
            // swizzled row per step) and adds w_v * sum into P[v] -- one
            // coalesced 128-byte reduction per run instead of one per edge
            float acc = 0.f;
            int cur = __shfl_sync(0xffffffffu, po, 0);
            float wcur = __shfl_sync(0xffffffffu, po_w, 0);
            const bool col_ok = c + lane < p.push_ld;
#pragma unroll 4
            for (int r = 0; r < 32; ++r) {
              const int v = __shfl_sync(0xffffffffu, po, r);
              const float wv = __shfl_sync(0xffffffffu, po_w, r);
              if (v != cur) {  // warp-uniform
                if (cur >= 0 && col_ok)
                  asm volatile("red.global.add.f32 [%0], %1;" ::"l"(p.push_out + (int64_t)cur * p.push_ld + c + lane),
                               "f"(acc * wcur)
                               : "memory");
                acc = 0.f;
                cur = v;
                wcur = wv;
              }
              float x;
              asm volatile("ld.shared.f32 %0, [%1];"
                           : "=f"(x)
                           : "r"(ob_u32 + r * 128 + ((((lane >> 2) ^ (r & 7))) << 4) + (lane & 3) * 4));
              acc += x;
            }
            if (cur >= 0 && col_ok)
              asm volatile("red.global.add.f32 [%0], %1;" ::"l"(p.push_out + (int64_t)cur * p.push_ld + c + lane),
                           "f"(acc * wcur)
                           : "memory");
          }
          if (push) {
            // P[v][c .. c+32) += w_v * Y[u][c .. c+32) for every in-edge
            // (v, u): four edges per instruction, eight lanes x 16 B = the
            // 128-byte row piece of one edge (coalesced L2 reductions)
            const int j4 = lane >> 3, qq = lane & 7;
            for (int p0 = 0; p0 < pe_total; p0 += 4) {
              const int pidx = p0 + j4;
              int vr = 0;
              float w = 0.f;
              if (p0 < 128) {
                const int slot = p0 >> 5;  // warp-uniform (p0 is a multiple of 4)
                const int src = pidx & 31;
                const int vk = slot == 0 ? pv[0] : slot == 1 ? pv[1] : slot == 2 ? pv[2] : pv[3];
                const float wk = slot == 0 ? pw[0] : slot == 1 ? pw[1] : slot == 2 ? pw[2] : pw[3];
                vr = __shfl_sync(0xffffffffu, vk, src);
                w = __shfl_sync(0xffffffffu, wk, src);
              } else {  // beyond the cached edges (hub rows): resolve on the fly
                int r = 0;
                for (int b = 16; b; b >>= 1) {
                  const int cand = r + b;
                  if (__shfl_sync(0xffffffffu, pe_incl, cand - 1) <= pidx) r = cand;
                }
                const int eb = __shfl_sync(0xffffffffu, pe_beg, r), ex = __shfl_sync(0xffffffffu, pe_excl, r);
                if (pidx < pe_total) {
                  const int v = __ldg(p.push_dst + eb + (pidx - ex));
                  vr = v | (r << 26);
                  w = 1.f;
                  if (p.push_mean) {
                    const int cv = __ldg(p.push_indptr + v + 1) - __ldg(p.push_indptr + v);
                    w = cv ? 1.f / (float)cv : 0.f;
                  }
                }
              }
              if (pidx < pe_total && c + 4 * qq < p.push_ld) {
                const int r = vr >> 26, v = vr & ((1 << 26) - 1);
                float4 x;
                asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                             : "=f"(x.x), "=f"(x.y), "=f"(x.z), "=f"(x.w)
                             : "r"(ob_u32 + r * 128 + ((qq ^ (r & 7)) << 4)));
                float* dst = p.push_out + (int64_t)v * p.push_ld + c + 4 * qq;
                asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst), "f"(x.x * w), "f"(x.y * w),
                             "f"(x.z * w), "f"(x.w * w)
                             : "memory");
              }
            }
          }
        }
        tc_before();
        __syncwarp();
        if (lane == 0) {  // one arrive per epilogue warp (PAIR: on the leader's barrier)
          if (PAIR) mbar_arrive_remote(map_rank(&tempty[acc], 0));
          else mbar_arrive(&tempty[acc]);
        }
      }
      if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
  } else {
    // =============================== dW ===============================
    const int nkb = kb1 - kb0;
    const int ig = blockIdx.y;  // i-tile group
    const int ngroups = MT * 4 + BN / 32;  // 32-column transposer work units
    if (warp == 0) {
      // gather4 (p.x1_rows): lanes 0..3 load graph rows 4l..4l+3 of each
      // k-block's X1 tiles, their indices fetched one k-block ahead; rows
      // >= M read table row 0 (the transposers zero them)
      const bool g4 = p.x1_rows != nullptr;
      auto rows4 = [&](int i, int (&r4)[4]) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int m = (kb0 + i) * DW_KR + 4 * lane + j;
          r4[j] = (i < nkb && m < M) ? __ldg(p.x1_rows + m) : 0;
        }
      };
      int rc[4] = {0, 0, 0, 0}, rn[4] = {0, 0, 0, 0};
      if (g4 && lane < 4) rows4(0, rc);
      if (lane == 0 || (g4 && lane < 4)) {
        for (int i = 0; i < nkb; ++i) {
          const int s = i % S;
          if (g4) rows4(i + 1, rn);
          uint8_t* sa = smem + (size_t)s * stage_bytes;
          const int row = (kb0 + i) * DW_KR;
          if (lane == 0) {
            if (i >= S) mbar_wait(&empty[s], ((i / S) & 1) ^ 1);
            uint32_t bytes = (uint32_t)b_bytes;
            for (int mt = 0; mt < MT; ++mt)
              if ((ig * MT + mt) * 4 < p.ablocks) bytes += DW_KR * BM * 4;
            mbar_arrive_tx(&full[s], bytes);
          }
          if (g4) __syncwarp(0xfu);
          for (int mt = 0; mt < MT; ++mt) {
            const int blk = (ig * MT + mt) * 4;  // first 32-wide i block of this 128-row tile
            if (blk >= p.ablocks) continue;
            uint8_t* dst = sa + mt * (DW_KR * BM * 4);
            if (blk < p.nkb1) {
              if (g4) tma_gather4(dst + lane * 4 * BM * 4, &p.ta1, blk * 32, rc[0], rc[1], rc[2], rc[3], &full[s]);
              else tma_load_2d(dst, &p.ta1, blk * 32, row, &full[s]);
            } else if (lane == 0) {
              tma_load_2d(dst, &p.ta2, (blk - p.nkb1) * 32, row, &full[s]);
            }
          }
          if (lane == 0) {
            tma_load_2d(sa + a_bytes, &p.tb, 0, row, &full[s]);
            if (p.mask) tma_load_2d(sa + a_bytes + g_bytes, &p.th, 0, row, &full[s]);
          }
#pragma unroll
          for (int j = 0; j < 4; ++j) rc[j] = rn[j];
        }
      }
    } else if (warp == 1) {
      // kind::tf32 accepts K-major operands only (an MN-major tf32 operand
      // yields zeros on sm_100a -- tools/umma_probe.cu), so the MMA reads the
      // K-major tiles the transposer warps build from each staged block.
      if (lane == 0) {
        const uint32_t idesc = idesc_tf32((uint32_t)BN, false, false);
        for (int i = 0; i < nkb; ++i) {
          const int b = i & 1;
          mbar_wait(&kready[b], (i >> 1) & 1);
          tc_after();
          const uint32_t ka = smem_u32(kbuf + (size_t)b * kt_bytes), kbb = ka + MT * BM * 64;
#pragma unroll
          for (int mt = 0; mt < MT; ++mt) {
#pragma unroll
            for (int k = 0; k < DW_KR / 8; ++k) {
              mma_tf32(tmem + (uint32_t)(mt * BN), desc_sw(ka + mt * BM * 64 + k * 32, 512, 4),
                         desc_sw(kbb + k * 32, 512, 4), idesc, (i > 0 || k > 0) ? 1u : 0u);
            }
          }
          mma_commit(&kfree[b]);
        }
        if (nkb > 0) mma_commit(&tfull[0]);
        else mbar_arrive(&tfull[0]);
      }
      __syncwarp();
    } else {
      // ---- transposers: a 32-column group of a staged [16 x cols] box -> 32
      // K-major SW64 rows (one per feature / output column, 16 graph rows of
      // K).  Lane (rq, cq) = (lane / 8, lane % 8) owns the 4 x 4 block rows
      // 4rq.., columns 4cq..: four LDS.128 along the staged rows, a register
      // transpose, and four STS.128 into the K-major rows (one 16-byte chunk
      // of 4 graph rows each) -- 8 shared-memory instructions per lane for
      // 16 elements.  Graph rows >= M (stale tail) and features beyond the
      // operand become 0.  With p.mask the G group is multiplied by its ReLU
      // bits (one staged word per graph row) and each lane keeps the column
      // sums of its 4 G' columns (db), reduced over rq at the end.
      const int tw = warp - 2;  // 0..NE-1
      const int rq = lane >> 3, cq = lane & 7;
      float dbacc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
      for (int i = 0; i < nkb; ++i) {
        const int s = i % S, b = i & 1;
        mbar_wait(&full[s], (i / S) & 1);
        if (i >= 2) mbar_wait(&kfree[b], ((i >> 1) - 1) & 1);  // MMA done with tile b
        const int valid = min(DW_KR, M - (kb0 + i) * DW_KR);
        const uint8_t* st = smem + (size_t)s * stage_bytes;
        uint8_t* kt = kbuf + (size_t)b * kt_bytes;
#pragma unroll
        for (int jb = 0; jb < 2; ++jb) {
          const int gx = tw + jb * NE;
          if (gx >= ngroups) break;
          const bool is_a = gx < MT * 4;
          const bool loaded = !is_a || ((ig * MT + gx / 4) * 4 < p.ablocks);
          const float* src;
          int ld;
          if (is_a) {
            src = reinterpret_cast<const float*>(st + (gx / 4) * (DW_KR * BM * 4)) + (gx % 4) * 32 + 4 * cq;
            ld = BM;
          } else {
            src = reinterpret_cast<const float*>(st + a_bytes) + (gx - MT * 4) * 32 + 4 * cq;
            ld = BN;
          }
          float4 x[4];
          if (!is_a && p.g16) {  // bf16 G: four elements (8 bytes) per staged row, widened to fp32
            const uint2* src16 = reinterpret_cast<const uint2*>(
                reinterpret_cast<const __nv_bfloat16*>(st + a_bytes) + (gx - MT * 4) * 32 + 4 * cq);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const int r = 4 * rq + j;
              const uint2 q = (r < valid) ? src16[r * (BN / 4)] : make_uint2(0u, 0u);
              x[j] = make_float4(__uint_as_float(q.x << 16), __uint_as_float(q.x & 0xFFFF0000u),
                                 __uint_as_float(q.y << 16), __uint_as_float(q.y & 0xFFFF0000u));
            }
          } else {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const int r = 4 * rq + j;
              x[j] = (loaded && r < valid) ? *reinterpret_cast<const float4*>(src + r * ld)
                                           : make_float4(0.f, 0.f, 0.f, 0.f);
            }
          }
          if (!is_a && p.mask) {
            const uint32_t* wb = reinterpret_cast<const uint32_t*>(st + a_bytes + g_bytes) + (gx - MT * 4);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const uint32_t w = wb[(4 * rq + j) * p.nwp] >> (4 * cq);
              if (!(w & 1u)) x[j].x = 0.f;
              if (!(w & 2u)) x[j].y = 0.f;
              if (!(w & 4u)) x[j].z = 0.f;
              if (!(w & 8u)) x[j].w = 0.f;
            }
          }
          if (!is_a && (p.mask || p.dbsum)) {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              dbacc[jb][0] += x[j].x;
              dbacc[jb][1] += x[j].y;
              dbacc[jb][2] += x[j].z;
              dbacc[jb][3] += x[j].w;
            }
          }
          const int krow0 = (is_a ? gx * 32 : MT * BM + (gx - MT * 4) * 32) + 4 * cq;
          const uint32_t kt_u32 = smem_u32(kt);
          // Store q writes feature (K-major row) krow0 + ((q + cq/2) & 3): the
          // per-lane rotation spreads each 8-lane phase of the STS.128 over
          // both row parities and all four SW64 chunks, i.e. all 32 banks
          // (one wavefront per phase; without it 8 lanes of a phase share 8
          // banks -- 4x the store wavefronts, measured 57% of the shared pipe)
          const int rot = cq >> 1;
          const bool r1 = rot & 1, r2 = rot & 2;
          float y[4][4];  // y[j][q] = component (q + rot) & 3 of x[j] (branch-free selects)
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float a = r1 ? x[j].y : x[j].x, b = r1 ? x[j].z : x[j].y;
            const float c = r1 ? x[j].w : x[j].z, e = r1 ? x[j].x : x[j].w;
            y[j][0] = r2 ? c : a;
            y[j][1] = r2 ? e : b;
            y[j][2] = r2 ? a : c;
            y[j][3] = r2 ? b : e;
          }
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int krow = krow0 + ((q + rot) & 3);
            st_shared_v4(kt_u32 + (uint32_t)krow * 64 + ((rq ^ ((krow >> 1) & 3)) << 4), y[0][q], y[1][q], y[2][q],
                         y[3][q]);
          }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // every writer, then one arrive per warp
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&empty[s]);   // staging stage s may be refilled
          mbar_arrive(&kready[b]);  // K-major tile b ready for the MMA
        }
      }
      if ((p.mask || p.dbsum) && ig == 0) {
#pragma unroll
        for (int jb = 0; jb < 2; ++jb) {
          const int gx = tw + jb * NE;
#pragma unroll
          for (int ci = 0; ci < 4; ++ci) {
            float v = dbacc[jb][ci];
            v += __shfl_xor_sync(0xffffffffu, v, 8);
            v += __shfl_xor_sync(0xffffffffu, v, 16);
            dbacc[jb][ci] = v;
          }
          if (gx >= MT * 4 && gx < ngroups && rq == 0) {
            const int col = (gx - MT * 4) * 32 + 4 * cq;
#pragma unroll
            for (int ci = 0; ci < 4; ++ci)
              if (col + ci < p.N) atomicAdd(p.db + col + ci, dbacc[jb][ci]);
          }
        }
      }
      mbar_wait(&tfull[0], 0);
      tc_after();
      const int q = warp & 3;
      const int half = (warp - 2) >> 2;
      const int row = q * 32 + lane;
      // split-K partial sums go straight into dW with vector float atomics
      // (red.global.add): row i' of the [X1 blocks | X2 blocks] space is
      // weight row k = i' (X1) or K1 + i' - 32*nkb1 (X2); padding rows skip.
      // (The backward's dH is accumulated with atomics too, so dW has no
      // fixed summation order to preserve.)
      for (int mt = 0; mt < MT && nkb > 0; ++mt) {
        const int irow = (ig * MT + mt) * BM + row;
        int k = -1;
        if (irow < 32 * p.nkb1) {
          if (irow < p.K1) k = irow;
        } else if (p.two && irow - 32 * p.nkb1 < p.K1) {
          k = p.K1 + irow - 32 * p.nkb1;
        }
        float* dst = p.dW + (int64_t)(k < 0 ? 0 : k) * p.N;
        for (int c = half * 32; c < BN; c += 64) {
          float v[32];
          tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(mt * BN + c), v);
          if (k < 0) continue;
          if ((p.N & 3) == 0) {
#pragma unroll
            for (int j = 0; j < 32; j += 4)
              if (c + j < p.N) atomicAdd(reinterpret_cast<float4*>(dst + c + j), make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]));
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (c + j < p.N) atomicAdd(dst + c + j, v[j]);
          }
        }
      }
    }
  }
  tc_before();
  __syncthreads();
  if (PAIR) cluster_sync_all();  // both CTAs done with the pair's TMEM and barriers
  if (warp == 1) {
    __syncwarp();
    tc_after();
    if (PAIR)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(ncols) : "memory");
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(ncols) : "memory");
  }
  if (dyn && threadIdx.x == 0) sched_done(p.sched);
}

// --------------------------------------------------------- prep kernels
// fwd B image: Bt[n][k'] (Npad x Kp, fp32, K-major), k' = kb*32 + c over
// [X1 blocks | X2 blocks]: k' < 32*nkb1 -> W row k' (valid < K1), else
// W row K1 + (k' - 32*nkb1) (valid < K1).
__global__ void k_bt_fwd(const float* __restrict__ W, int K1, int nkb1, int two, int N, int Npad, int Kp, float* Bt) {
  GNNV_PDL_ENTRY();
  const int total = Npad * Kp;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
    const int n = t / Kp, kp = t - n * Kp;
    int k = -1;
    if (kp < 32 * nkb1) {
      if (kp < K1) k = kp;
    } else if (two) {
      const int kk = kp - 32 * nkb1;
      if (kk < K1) k = K1 + kk;
    }
    Bt[t] = (k >= 0 && n < N) ? W[(int64_t)k * N + n] : 0.f;
  }
}
// bf16 fwd B image: Bt16[n][kp] (Npad x Kp), 64-element k-blocks: X1's
// nkb1 blocks then X2's; columns past K1 in each part are zero (X1's bf16
// copy may carry a ones column there)
__global__ void k_bt_fwd16(const float* __restrict__ W, int K1, int nkb1, int two, int N, int Npad, int Kp,
                           __nv_bfloat16* Bt) {
  GNNV_PDL_ENTRY();
  const int total = Npad * Kp;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
    const int n = t / Kp, kp = t - n * Kp;
    int k = -1;
    if (kp < 64 * nkb1) {
      if (kp < K1) k = kp;
    } else if (two) {
      const int kk = kp - 64 * nkb1;
      if (kk < K1) k = K1 + kk;
    }
    Bt[t] = __float2bfloat16_rn((k >= 0 && n < N) ? W[(int64_t)k * N + n] : 0.f);
  }
}
// bf16 dX B image: as k_bt_dx, bf16 (64-element k-blocks)
__global__ void k_bt_dx16(const float* __restrict__ W, int K1, int ld1, int ld2, int two, int N, int NCpad, int Kp,
                          __nv_bfloat16* Bd) {
  GNNV_PDL_ENTRY();
  const int total = NCpad * Kp;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
    const int j = t / Kp, k = t - j * Kp;
    int r = -1;
    if (j < ld1) {
      if (j < K1) r = j;
    } else if (two && j - ld1 < ld2 && j - ld1 < K1) {
      r = K1 + (j - ld1);
    }
    Bd[t] = __float2bfloat16_rn((r >= 0 && k < N) ? W[(int64_t)r * N + k] : 0.f);
  }
}
// dX B image: Bd[j][k] (NCpad x Kp): j over [0, ld1) -> W row j (< K1),
// [ld1, ld1+ld2) -> W row K1 + (j - ld1); k < N.
__global__ void k_bt_dx(const float* __restrict__ W, int K1, int ld1, int ld2, int two, int N, int NCpad, int Kp,
                        float* Bd) {
  GNNV_PDL_ENTRY();
  const int total = NCpad * Kp;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
    const int j = t / Kp, k = t - j * Kp;
    int r = -1;
    if (j < ld1) {
      if (j < K1) r = j;
    } else if (two && j - ld1 < ld2 && j - ld1 < K1) {
      r = K1 + (j - ld1);
    }
    Bd[t] = (r >= 0 && k < N) ? W[(int64_t)r * N + k] : 0.f;
  }
}
// ------------------------------------------------------ host helpers
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    GNNV_TRY_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    GNNV_REQUIRE(p && q == cudaDriverEntryPointSuccess, GNNV_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
  }
  return fn;
}

// 2-D fp32 row-major tensor [rows x cols] with row stride ld (floats); box
// [box_rows x 32 cols], 128B swizzle, out-of-range elements read as zero.
// bf16 2-D map, no swizzle (the dW's G operand when it is a bf16 copy)
static CUtensorMap make_map16(const void* base, int64_t rows, int64_t cols, int64_t ld, int box_rows, int box_cols) {
  CUtensorMap m;
  const cuuint64_t dims[2] = {(cuuint64_t)std::max<int64_t>(cols, 1), (cuuint64_t)std::max<int64_t>(rows, 1)};
  const cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
  const cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  GNNV_REQUIRE(r == CUDA_SUCCESS, GNNV_ERR_CUDA, "cuTensorMapEncodeTiled (bf16) failed (alignment/stride)");
  return m;
}

// bf16 2-D map with 64-element (128-byte) x box_rows boxes and the 128-byte swizzle (UMMA operands)
static CUtensorMap make_map16_sw(const void* base, int64_t rows, int64_t cols, int64_t ld, int box_rows = 64) {
  CUtensorMap m;
  const cuuint64_t dims[2] = {(cuuint64_t)std::max<int64_t>(cols, 1), (cuuint64_t)std::max<int64_t>(rows, 1)};
  const cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
  const cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  GNNV_REQUIRE(r == CUDA_SUCCESS, GNNV_ERR_CUDA, "cuTensorMapEncodeTiled (bf16 SW128) failed (alignment/stride)");
  return m;
}

static CUtensorMap make_map(const float* base, int64_t rows, int64_t cols, int64_t ld, int box_rows,
                            int box_cols = 32, bool swizzle = true) {
  CUtensorMap m;
  const cuuint64_t dims[2] = {(cuuint64_t)std::max<int64_t>(cols, 1), (cuuint64_t)std::max<int64_t>(rows, 1)};
  const cuuint64_t strides[1] = {(cuuint64_t)ld * sizeof(float)};
  const cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)base, dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE,
                           swizzle ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  GNNV_REQUIRE(r == CUDA_SUCCESS, GNNV_ERR_CUDA, "cuTensorMapEncodeTiled failed (alignment/stride)");
  return m;
}

struct Arena {
  void* buf = nullptr;
  size_t cap = 0;
  void* get(size_t bytes, cudaStream_t s) {
    if (bytes > cap) {
      if (buf) {
        GNNV_TRY_CUDA(cudaStreamSynchronize(s));
        dfree(buf);
      }
      cap = std::max(bytes, (size_t)4 << 20);
      buf = dmalloc(cap, "tf32 GEMM workspace");
    }
    return buf;
  }
};
static Arena g_img;
static Arena g_dwpart;  // gemm_dw16's per-CTA slices
static Arena g_dbpart;  // its G conversion's per-block column sums

// bres_nkb > 0: the forward's W^T resident (bres_nkb k-blocks of BN x 128B), stages of A only
static size_t smem_bytes(int mode, int BN, int mask, int nwp, bool pair = false, int g16 = 0, int bres_nkb = 0) {
  const int S = mode == MODE_DW ? (g16 ? DW_STAGES16 : DW_STAGES) : pair ? PAIR_STAGES : FWD_STAGES;
  const int a = mode == MODE_DW ? DW_MT * DW_KR * BM * 4 : BM * BKB;
  const int b = mode == MODE_DW ? DW_KR * BN * (g16 ? 2 : 4) + (mask ? DW_KR * nwp * 4 : 0)
                : bres_nkb ? 0 : (pair ? BN / 2 : BN) * BKB;
  const int k = mode == MODE_DW ? 2 * (DW_MT * BM + BN) * 64 : NE * 4096 * (pair ? PAIR_OB : 1);
  return (size_t)bres_nkb * BN * BKB + (((size_t)S * (a + b) + 1023) & ~(size_t)1023) + k + 8 * (2 * S + 8 + 8) +
         32 + 16 + 16 + 1024;
}

template <int MODE>
static void launch(const Params& p, dim3 grid, cudaStream_t s) {
  static size_t attr = 0;  // dynamic smem opt-in, raised to the largest request seen
  const size_t bytes = smem_bytes(MODE, p.BN, p.mask, p.nwp, false, p.g16, MODE == MODE_FWD && p.bres ? p.nkb : 0);
  if (bytes > attr) {
    GNNV_TRY_CUDA(cudaFuncSetAttribute(k_tma_gemm<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    attr = bytes;
  }
  launch_k(k_tma_gemm<MODE>, grid, NTHREADS, bytes, s, p);
  GNNV_CHECK_LAUNCH();
}

// the CTA-pair forward GEMM: clusters of 2 along x
static void launch_pair(const Params& p, int pairs, cudaStream_t s) {
  static size_t attr = 0;
  const size_t bytes = smem_bytes(MODE_FWD, p.BN, p.mask, p.nwp, true);
  if (bytes > attr) {
    GNNV_TRY_CUDA(cudaFuncSetAttribute(k_tma_gemm<MODE_FWD, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)bytes));
    attr = bytes;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(2 * pairs));
  cfg.blockDim = dim3(NTHREADS);
  cfg.dynamicSmemBytes = bytes;
  cfg.stream = s;
  cudaLaunchAttribute attrs[2];
  attrs[0].id = cudaLaunchAttributeClusterDimension;
  attrs[0].val.clusterDim.x = 2;
  attrs[0].val.clusterDim.y = 1;
  attrs[0].val.clusterDim.z = 1;
  int na = 1;
  if (pdl_enabled()) {
    attrs[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attrs[1].val.programmaticStreamSerializationAllowed = 1;
    na = 2;
  }
  cfg.attrs = attrs;
  cfg.numAttrs = na;
  GNNV_TRY_CUDA(cudaLaunchKernelEx(&cfg, k_tma_gemm<MODE_FWD, true>, p));
  GNNV_CHECK_LAUNCH();
}

static int rup(int x, int m) { return (x + m - 1) / m * m; }

// a scheduler slot for the next fwd/dX launch (ring of 4096; a slot is reset
// by the last CTA of the launch that used it).  GNNV_STATIC_TILES=1: the
// static round robin instead.
static unsigned int* sched_slot();
static unsigned int* next_sched() {
  if (env_on("GNNV_STATIC_TILES")) return nullptr;
  return sched_slot();
}
static unsigned int* sched_slot() {
  static unsigned int* base = nullptr;
  static unsigned slot = 0;
  if (!base) {
    void* p = nullptr;
    GNNV_TRY_CUDA(cudaGetSymbolAddress(&p, g_sched));
    base = static_cast<unsigned int*>(p);
  }
  return base + 2 * (slot++ % 4096);
}

// ------------------------------------------------ dW over bf16 operands
// The layer-1 weight gradient of the trainer with bf16 intermediates and
// the bf16 table (readings Q30/Q31): dW = [X16 | A16]^T G16 with all three
// operands bf16 in HBM.  kind::f16 accepts MN-major operands (measured with
// tools/umma_probe.cu: bf16 MN/MN exact, tf32 MN-major all zeros), so the
// TMA-staged row-major boxes feed the MMA directly -- no transposer warps:
// A = X^T with M = features (two 64-feature SW128 boxes per 128-row tile,
// 8 KB apart = LBO) and K = graph rows (8-row groups 1024 B apart = SBO),
// B = G with N = output columns (BN/64 boxes).  64 graph rows per k-block
// (four K = 16 MMAs per tile), split-K over graph rows across the grid,
// partial sums added into dW with red.global.add.  X16's column K1 holds
// 1.0, so row K1 of the first tile is colsum(G) = db.  The MMA warp zeroes
// the rows of a ragged last k-block past M in shared memory (rows past the
// buffers' max_M arrive zero-filled from TMA).
constexpr int DW16_KR = 64;
constexpr int DW16_STAGES = 3;
constexpr int DW16_CHUNK = 4;  // k-blocks per scheduled chunk
constexpr int DW16_BOX = DW16_KR * 128;  // one 64-row x 64-bf16 box, bytes

__device__ __forceinline__ uint64_t desc_mn128(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;  // SWIZZLE_128B
  return d;
}

// one 128-feature M tile: features [col0, col0 + 128) of a bf16 source
// (two 64-feature boxes); TMEM lane r -> dW row out_row0 + r for r <
// out_rows, lane db_row -> db (the source's ones column; -1: none)
struct Dw16Tile {
  CUtensorMap map;
  int col0, out_row0, out_rows, db_row;
};
struct Dw16Params {
  Dw16Tile tile[4];      // CTA group g = blockIdx.y takes tiles 2g and 2g + 1
  CUtensorMap tg;        // G16 [rows x ldg], boxes of 64 x 64, SW128
  const int32_t* dM;
  unsigned int* sched[2];  // each group's chunk counter (g_sched slots)
  int N, BN;
  float *dW, *db;
  // CTA x's sums go to part[x][row][N] (row = dW row, db at prow - 1) with
  // plain stores; k_dw16_reduce adds the CTAs' slices in a fixed order
  float* part;
  int prow;
};

__global__ void __launch_bounds__(NTHREADS, 1) k_tma_dw16(const __grid_constant__ Dw16Params p) {
  GNNV_PDL_ENTRY();
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  constexpr int S = DW16_STAGES;
  const int BN = p.BN;
  const int nb = BN / 64;
  const int a_bytes = 4 * DW16_BOX;  // two tiles (X, A) x two 64-feature boxes
  const int stage_bytes = a_bytes + nb * DW16_BOX;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)S * stage_bytes);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;
  int32_t* s_kb = reinterpret_cast<int32_t*>(tfull + 1);  // [S]: the k-block in each stage, -1 = no more
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(s_kb + S);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int M = *p.dM;
  const int nkbm = (M + DW16_KR - 1) / DW16_KR;
  const int nchunks = (nkbm + DW16_CHUNK - 1) / DW16_CHUNK;
  const int grp = blockIdx.y;
  const Dw16Tile& T0 = p.tile[2 * grp];
  const Dw16Tile& T1 = p.tile[2 * grp + 1];
  unsigned int* sched = p.sched[grp];
  // chunks of DW16_CHUNK k-blocks: chunk blockIdx.x first, then claimed from
  // the launch's counter -- a CTA slowed by a co-resident kernel (the Eq.4
  // prefetch) takes fewer; every CTA keeps its sums in TMEM and flushes once
  const bool any = (int)blockIdx.x < nchunks;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch(&T0.map);
    tma_prefetch(&T1.map);
    tma_prefetch(&p.tg);
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(s_tmem)), "r"(2 * 256)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_before();
  __syncthreads();
  tc_after();
  const uint32_t tmem = *s_tmem;
  if (warp == 0) {
    if (lane == 0) {
      int i = 0;
      for (int c = blockIdx.x; c < nchunks; c = (int)gridDim.x + (int)atomicAdd(sched, 1u)) {
        const int kb_end = min(nkbm, (c + 1) * DW16_CHUNK);
        for (int kb = c * DW16_CHUNK; kb < kb_end; ++kb, ++i) {
          const int s = i % S;
          uint8_t* st = smem + (size_t)s * stage_bytes;
          const int row = kb * DW16_KR;
          if (i >= S) mbar_wait(&empty[s], ((i / S) & 1) ^ 1);
          s_kb[s] = kb;
          mbar_arrive_tx(&full[s], (uint32_t)stage_bytes);
          tma_load_2d(st, &T0.map, T0.col0, row, &full[s]);
          tma_load_2d(st + DW16_BOX, &T0.map, T0.col0 + 64, row, &full[s]);
          tma_load_2d(st + 2 * DW16_BOX, &T1.map, T1.col0, row, &full[s]);
          tma_load_2d(st + 3 * DW16_BOX, &T1.map, T1.col0 + 64, row, &full[s]);
          for (int j = 0; j < nb; ++j) tma_load_2d(st + a_bytes + j * DW16_BOX, &p.tg, 64 * j, row, &full[s]);
        }
      }
      const int s = i % S;  // end marker
      if (i >= S) mbar_wait(&empty[s], ((i / S) & 1) ^ 1);
      s_kb[s] = -1;
      mbar_arrive(&full[s]);
    }
    __syncwarp();
  } else if (warp == 1) {
    // D f32, A = B = bf16, both MN-major, N = BN, M = 128
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | (1u << 16) |
                           ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
    int i = 0;
    for (;; ++i) {
      const int s = i % S;
      mbar_wait(&full[s], (i / S) & 1);
      const int kb = s_kb[s];
      if (kb < 0) break;
      const int valid = M - kb * DW16_KR;
      if (valid < DW16_KR) {  // ragged last k-block: rows M.. of every box hold stale data -> zero them
        uint8_t* st = smem + (size_t)s * stage_bytes;
        const int per_box = (DW16_KR - valid) * 8;  // 16-byte chunks
        for (int q = lane; q < (4 + nb) * per_box; q += 32) {
          const int box = q / per_box, k = q - box * per_box;
          *reinterpret_cast<uint4*>(st + (size_t)box * DW16_BOX + (size_t)valid * 128 + (size_t)k * 16) =
              make_uint4(0u, 0u, 0u, 0u);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      }
      __syncwarp();
      tc_after();
      if (lane == 0) {
        const uint32_t a0 = smem_u32(smem + (size_t)s * stage_bytes), b0 = a0 + a_bytes;
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
          for (int ks = 0; ks < DW16_KR / 16; ++ks)
            mma_f16(tmem + (uint32_t)(mt * BN), desc_mn128(a0 + mt * 2 * DW16_BOX + ks * 2048, DW16_BOX, 1024),
                    desc_mn128(b0 + ks * 2048, DW16_BOX, 1024), idesc, (i > 0 || ks > 0) ? 1u : 0u);
        mma_commit(&empty[s]);
      }
      __syncwarp();
    }
    if (lane == 0) {
      if (i > 0) mma_commit(tfull);
      else mbar_arrive(tfull);
    }
    __syncwarp();
  } else if (any || p.part) {
    if (any) {
      mbar_wait(tfull, 0);
      tc_after();
    }
    const int q = warp & 3;
    const int half = (warp - 2) >> 2;
    const int r = q * 32 + lane;  // TMEM lane = row of the 128-row tile
    for (int mt = 0; mt < 2; ++mt) {
      const Dw16Tile& T = mt ? T1 : T0;
      float* dst = nullptr;
      if (p.part) {  // this CTA's slice (a CTA without chunks writes zeros)
        float* slice = p.part + (int64_t)blockIdx.x * p.prow * p.N;
        if (r < T.out_rows) dst = slice + (int64_t)(T.out_row0 + r) * p.N;
        else if (r == T.db_row) dst = slice + (int64_t)(p.prow - 1) * p.N;
      } else {
        if (r < T.out_rows) dst = p.dW + (int64_t)(T.out_row0 + r) * p.N;
        else if (r == T.db_row) dst = p.db;  // the source's ones column
      }
      for (int c = half * 32; c < BN; c += 64) {
        float v[32];
        if (any) tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(mt * BN + c), v);
        else
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = 0.f;
        if (!dst) continue;
        if (p.part) {
#pragma unroll
          for (int j = 0; j < 32; j += 4)
            if (c + j < p.N) __stcg(reinterpret_cast<float4*>(dst + c + j), make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]));
        } else {
#pragma unroll
          for (int j = 0; j < 32; j += 4)
            if (c + j < p.N)
              atomicAdd(reinterpret_cast<float4*>(dst + c + j), make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]));
        }
      }
    }
  }
  tc_before();
  __syncthreads();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * 256) : "memory");
  if (threadIdx.x == 0) {  // the group's last CTA resets its counter
    __threadfence();
    if (atomicAdd(sched + 1, 1u) == gridDim.x - 1) {
      sched[0] = 0u;
      sched[1] = 0u;
      __threadfence();
    }
  }
}

// G (fp32, already masked) -> its bf16 copy, and per-block column sums
// (db's partials, summed by k_dw16_reduce in block order): 4 rows of 64
// float4 columns per pass, four rows per thread in flight
__global__ void __launch_bounds__(256) k_g16_colsum(const float* __restrict__ G, int ldg, const int32_t* d_M, int N,
                                                    __nv_bfloat16* __restrict__ G16, int ld16, float* __restrict__ dbp) {
  GNNV_PDL_ENTRY();
  __shared__ float4 s_acc[256];
  const int M = *d_M;
  const int n4 = N >> 2;  // <= 64
  const int rg = threadIdx.x >> 6, c4 = threadIdx.x & 63;
  const int per = (M + gridDim.x - 1) / gridDim.x;
  const int r0 = min(M, (int)blockIdx.x * per), r1 = min(M, r0 + per);
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  if (c4 < n4) {
    for (int r = r0 + rg; r < r1; r += 16) {
      float4 g[4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        g[u] = r + 4 * u < r1 ? __ldg(reinterpret_cast<const float4*>(G + (int64_t)(r + 4 * u) * ldg) + c4)
                              : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (r + 4 * u >= r1) continue;
        const __nv_bfloat162 lo = __floats2bfloat162_rn(g[u].x, g[u].y), hi = __floats2bfloat162_rn(g[u].z, g[u].w);
        reinterpret_cast<uint2*>(G16 + (int64_t)(r + 4 * u) * ld16)[c4] =
            make_uint2(*reinterpret_cast<const uint32_t*>(&lo), *reinterpret_cast<const uint32_t*>(&hi));
        acc.x += g[u].x; acc.y += g[u].y; acc.z += g[u].z; acc.w += g[u].w;
      }
    }
  }
  s_acc[threadIdx.x] = acc;
  __syncthreads();
  if (rg == 0 && c4 < n4) {
    float4 t = s_acc[c4];
    for (int q = 1; q < 4; ++q) {
      const float4 u = s_acc[q * 64 + c4];
      t.x += u.x; t.y += u.y; t.z += u.z; t.w += u.w;
    }
    reinterpret_cast<float4*>(dbp)[(int64_t)blockIdx.x * n4 + c4] = t;
  }
}

// dW (and db) = the CTAs' slices summed in a fixed order (deterministic): a
// block takes 32 float4 columns-chunks x 8 slice groups; thread (e, g) sums
// slices g, g + 8, ... of element e (four loads in flight), then the 8 group
// sums are added in group order through shared memory
__global__ void __launch_bounds__(256) k_dw16_reduce(const float* __restrict__ part, int splits, int prow, int N,
                                                     int has_db, float* __restrict__ dW, float* __restrict__ db,
                                                     const float* __restrict__ dbp, int ndbp) {
  GNNV_PDL_ENTRY();
  __shared__ float4 s_acc[8][33];
  const int n4 = N >> 2;
  const int64_t total = (int64_t)prow * n4, slice4 = (int64_t)prow * n4;
  const int e = threadIdx.x & 31, g = threadIdx.x >> 5;
  for (int64_t t0 = blockIdx.x * 32ll; t0 < total; t0 += (int64_t)gridDim.x * 32) {
    const int64_t t = t0 + e;
    const int row = t < total ? (int)(t / n4) : 0;
    const bool dbrow = t < total && row == prow - 1;
    const float4* P = reinterpret_cast<const float4*>(dbrow && dbp ? dbp : part);
    const int64_t stride = dbrow && dbp ? n4 : slice4;
    const int64_t off = dbrow && dbp ? t - (int64_t)row * n4 : t;
    const int cnt = dbrow && dbp ? ndbp : splits;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    if (t < total && (!dbrow || has_db)) {
      int sidx = g;
      for (; sidx + 24 < cnt; sidx += 32) {
        const float4 a = __ldcg(P + (int64_t)sidx * stride + off), b = __ldcg(P + (int64_t)(sidx + 8) * stride + off);
        const float4 c = __ldcg(P + (int64_t)(sidx + 16) * stride + off), d = __ldcg(P + (int64_t)(sidx + 24) * stride + off);
        acc.x += a.x; acc.y += a.y; acc.z += a.z; acc.w += a.w;
        acc.x += b.x; acc.y += b.y; acc.z += b.z; acc.w += b.w;
        acc.x += c.x; acc.y += c.y; acc.z += c.z; acc.w += c.w;
        acc.x += d.x; acc.y += d.y; acc.z += d.z; acc.w += d.w;
      }
      for (; sidx < cnt; sidx += 8) {
        const float4 a = __ldcg(P + (int64_t)sidx * stride + off);
        acc.x += a.x; acc.y += a.y; acc.z += a.z; acc.w += a.w;
      }
    }
    s_acc[g][e] = acc;
    __syncthreads();
    if (g == 0 && t < total && (!dbrow || has_db)) {
      float4 r = s_acc[0][e];
#pragma unroll
      for (int q = 1; q < 8; ++q) {
        const float4 u = s_acc[q][e];
        r.x += u.x; r.y += u.y; r.z += u.z; r.w += u.w;
      }
      float4* out = dbrow ? reinterpret_cast<float4*>(db) + (t - (int64_t)row * n4) : reinterpret_cast<float4*>(dW) + t;
      *out = r;
    }
    __syncthreads();
  }
}

}  // namespace tma

bool gemm_fwd_tma(const GemmFwdArgs& a, cudaStream_t s) {
  using namespace tma;
  const int BN = rup(a.ldy, 16);
  if (BN > 256) return false;
  const bool f16 = a.X1_16 != nullptr;
  const int kc = f16 ? 2 * BK : BK;  // elements per k-block
  const int nkb1 = (a.K1 + kc - 1) / kc;
  const int nkb = a.X2 || (f16 && a.X2_16) ? 2 * nkb1 : nkb1;
  const int Kp = nkb * kc;
  void* Bt = g_img.get((size_t)BN * Kp * (f16 ? 2 : 4), s);
  if (f16)
    launch_k(k_bt_fwd16, std::min(1024, (BN * Kp + 255) / 256), 256, 0, s, a.W, a.K1, nkb1, a.X2_16 ? 1 : 0, a.N, BN,
             Kp, (__nv_bfloat16*)Bt);
  else
    launch_k(k_bt_fwd, std::min(1024, (BN * Kp + 255) / 256), 256, 0, s, a.W, a.K1, nkb1, a.X2 ? 1 : 0, a.N, BN, Kp,
             (float*)Bt);
  GNNV_CHECK_LAUNCH();
  Params p{};
  p.f16 = f16 ? 1 : 0;
  p.x1_rows = a.x1_rows;
  // CTA pairs (cta_group::2) with GNNV_GEMM_PAIR=1 (read per call).  Off by
  // default: measured on products, layer 1 179 -> 189-192 us (its tiles are
  // bound by the A operand's DRAM reads and the epilogue, not by the W^T
  // traffic the pair halves), layer 2 49 -> 46 us
  const bool pair = env_on("GNNV_GEMM_PAIR") && !a.x1_rows && !a.push_out && BN % 32 == 0 && !f16;
  if (f16) {
    GNNV_REQUIRE(!a.x1_rows && a.ld16in % 8 == 0 && a.ld16in >= a.K1, GNNV_ERR_PARAM,
                 "fwd: bf16 operands need plain rows with a stride (multiple of 8) covering K1");
    p.ta1 = make_map16_sw(a.X1_16, a.max_M, a.ld16in, a.ld16in, BM);
    p.ta2 = a.X2_16 ? make_map16_sw(a.X2_16, a.max_M, a.ld16in, a.ld16in, BM) : p.ta1;
    p.tb = make_map16_sw(Bt, BN, Kp, Kp, BN);
    p.two = a.X2_16 ? 1 : 0;
  } else {
    p.ta1 = a.x1_rows ? make_map(a.X1, a.x1_table_rows, a.K1, a.ld1, 1) : make_map(a.X1, a.max_M, a.K1, a.ld1, BM);
    p.ta2 = a.X2 ? make_map(a.X2, a.max_M, a.K1, a.ld2, BM) : p.ta1;
    p.tb = make_map((const float*)Bt, BN, Kp, Kp, pair ? BN / 2 : BN);
    p.two = a.X2 ? 1 : 0;
  }
  p.nkb1 = nkb1;
  p.nkb = nkb;
  p.BN = BN;
  p.n_ntiles = 1;
  p.dM = a.d_M;
  p.Y = a.Y;
  p.ldy = a.ldy;
  p.N = a.N;
  p.bias = a.bias;
  p.relu = a.relu ? 1 : 0;
  p.ty1 = make_map(a.Y, a.max_M, a.ldy, a.ldy, 32);
  p.bits = a.relu ? a.mask_bits : nullptr;
  p.bits_ld = a.mask_ld;
  p.push_colptr = a.push_colptr;
  p.push_dst = a.push_dst;
  p.push_indptr = a.push_indptr;
  p.push_out = a.push_out;
  p.push_ld = a.push_ld;
  p.push_mean = a.push_mean ? 1 : 0;
  p.keep_rows = a.keep_rows;
  p.push_owner = a.push_owner;
  p.y16 = static_cast<__nv_bfloat16*>(a.y16);
  p.ld16 = a.ld16;
  if (a.y16) p.ty16 = make_map16(a.y16, a.max_M, a.ld16, a.ld16, 32, 32);
  GNNV_REQUIRE(!a.y16 || (a.ld16 % 32 == 0 && a.ld16 >= a.N && a.keep_rows), GNNV_ERR_PARAM,
               "fwd: bf16 copy needs a row stride that is a multiple of 32 and the kept-row count");
  GNNV_REQUIRE(!a.push_out || (a.push_colptr && a.push_dst && a.push_indptr && a.keep_rows && a.push_ld % 4 == 0 &&
                               a.push_ld >= a.N),
               GNNV_ERR_PARAM, "fwd: incomplete fused-push arguments");
  // W^T resident in shared memory when it fits beside the A stages and the
  // epilogue buffers (layer 1 over [X16 | A16]: 4 k-blocks, 128 KB): each
  // tile then streams only its A rows instead of re-reading W^T from L2
  p.bres = f16 && !pair && !a.x1_rows && !env_on("GNNV_NO_BRES") &&
           smem_bytes(MODE_FWD, BN, 0, 0, false, 0, nkb) <= (size_t)227 * 1024;
  p.eppipe = !env_on("GNNV_NO_EPPIPE");
  p.sched = pair ? nullptr : next_sched();
  const int64_t tiles = ceil_div(std::max<int64_t>(a.max_M, 1), BM);
  if (pair) {
    launch_pair(p, (int)std::min<int64_t>(ceil_div(tiles, 2), num_sms() / 2), s);
    return true;
  }
  launch<MODE_FWD>(p, dim3((unsigned)std::min<int64_t>(tiles, num_sms())), s);
  return true;
}

bool gemm_dx_tma(const GemmDxArgs& a, cudaStream_t s) {
  using namespace tma;
  const int NC = a.Y2 ? a.ld1 + a.ld2 : a.ld1;
  const int ntl = (NC + 255) / 256;
  const int BN = rup((NC + ntl - 1) / ntl, 32);  // whole 32-column epilogue chunks
  const bool f16 = a.G16 != nullptr;
  const int kc = f16 ? 2 * BK : BK;
  const int nkb = (a.N + kc - 1) / kc;
  const int Kp = nkb * kc;
  const int NCpad = ntl * BN;
  void* Bd = g_img.get((size_t)NCpad * Kp * (f16 ? 2 : 4), s);
  if (f16)
    launch_k(k_bt_dx16, std::min(1024, (NCpad * Kp + 255) / 256), 256, 0, s, a.W, a.K1, a.ld1, a.ld2, a.Y2 ? 1 : 0, a.N,
             NCpad, Kp, (__nv_bfloat16*)Bd);
  else
    launch_k(k_bt_dx, std::min(1024, (NCpad * Kp + 255) / 256), 256, 0, s, a.W, a.K1, a.ld1, a.ld2, a.Y2 ? 1 : 0, a.N,
             NCpad, Kp, (float*)Bd);
  GNNV_CHECK_LAUNCH();
  Params p{};
  p.f16 = f16 ? 1 : 0;
  if (f16) {
    GNNV_REQUIRE(a.ldg16 % 8 == 0 && a.ldg16 >= a.N, GNNV_ERR_PARAM, "dX: the bf16 G stride must be a multiple of 8 >= N");
    p.ta1 = make_map16_sw(a.G16, a.max_M, a.N, a.ldg16, BM);
    p.tb = make_map16_sw(Bd, NCpad, Kp, Kp, BN);
  } else {
    p.ta1 = make_map(a.G, a.max_M, a.N, a.ldg, BM);
    p.tb = make_map((const float*)Bd, NCpad, Kp, Kp, BN);
  }
  p.ta2 = p.ta1;
  p.nkb1 = nkb;
  p.nkb = nkb;
  p.BN = BN;
  p.n_ntiles = ntl;
  p.dM = a.d_M;
  p.Y1 = a.Y1;
  p.Y2 = a.Y2;
  p.ld1 = a.ld1;
  p.ld2 = a.ld2;
  p.ty2 = a.Y2 ? make_map(a.Y2, a.max_M, a.ld2, a.ld2, 32) : CUtensorMap{};
  if (a.Y1_16) {  // Y1 as bf16 rows: plain stores from the epilogue (ty1 unused)
    GNNV_REQUIRE(a.ld1 % 32 == 0 && a.Y2, GNNV_ERR_PARAM, "dX: a bf16 Y1 needs ld1 % 32 == 0 and Y2");
    p.y1_16 = static_cast<__nv_bfloat16*>(a.Y1_16);
    p.ty16 = make_map16(a.Y1_16, a.max_M, a.ld1, a.ld1, 32, 32);
    if (a.Y2_16) {
      GNNV_REQUIRE(a.ld2 % 32 == 0, GNNV_ERR_PARAM, "dX: a bf16 Y2 needs ld2 % 32 == 0");
      p.y2_16 = static_cast<__nv_bfloat16*>(a.Y2_16);
      p.ty2_16 = make_map16(a.Y2_16, a.max_M, a.ld2, a.ld2, 32, 32);
    }
    p.ty1 = p.ty2;
  } else {
    p.ty1 = make_map(a.Y1, a.max_M, a.ld1, a.ld1, 32);
    if (!a.Y2) p.ty2 = p.ty1;
  }
  p.ybits = a.y1_bits;
  p.ybits_ld = a.y1_bits_ld;
  const int64_t tiles = ceil_div(std::max<int64_t>(a.max_M, 1), BM) * ntl;
  p.sched = next_sched();
  launch<MODE_DX>(p, dim3((unsigned)std::min<int64_t>(tiles, num_sms())), s);
  return true;
}


// dW; with a.mask_bits also the fused ReLU mask and db (else db comes from the
// column-sum kernel in layers.cu).
void gemm_dw16(const GemmDw16Args& a, cudaStream_t s) {
  using namespace tma;
  GNNV_REQUIRE(a.N % 64 == 0 && a.N <= 256 && a.ldg % 8 == 0 && a.ldg >= a.N, GNNV_ERR_UNSUPPORTED,
               "dw16: N % 64 == 0 and N <= 256, G stride a multiple of 8");
  Dw16Params p{};
  int nt = 0, rows = 0;
  bool has_db = false;
  for (const GemmDw16Src& sr : a.src) {
    if (!sr.p) continue;
    const int w1 = sr.width + (sr.ones ? 1 : 0);
    GNNV_REQUIRE(sr.ld % 8 == 0 && sr.ld >= w1 && nt + (w1 + 127) / 128 <= 4, GNNV_ERR_UNSUPPORTED,
                 "dw16: source strides multiples of 8 covering the width (+ ones), at most four 128-feature tiles");
    const CUtensorMap m = make_map16_sw(sr.p, a.max_M, sr.ld, sr.ld);
    for (int j = 0; 128 * j < w1; ++j) {
      Dw16Tile& T = p.tile[nt++];
      T.map = m;
      T.col0 = 128 * j;
      T.out_row0 = sr.out_row0 + 128 * j;
      T.out_rows = std::max(0, std::min(128, sr.width - 128 * j));
      T.db_row = (sr.ones && sr.width >= 128 * j && sr.width < 128 * j + 128) ? sr.width - 128 * j : -1;
    }
    rows += sr.width;
    has_db = has_db || sr.ones;
  }
  GNNV_REQUIRE(nt > 0 && (!has_db || a.db) && (!a.G32 || (a.db && !has_db && a.ldg32 % 4 == 0)) &&
                   (!a.dbp || (a.db && !has_db && !a.G32)),
               GNNV_ERR_PARAM, "dw16: no source, or an inconsistent db source (ones column / G32 / partials)");
  if (nt & 1) {  // the last group's second tile: stages the same boxes, stores nothing
    p.tile[nt] = p.tile[nt - 1];
    p.tile[nt].out_rows = 0;
    p.tile[nt].db_row = -1;
    ++nt;
  }
  const int groups = nt / 2;
  p.tg = make_map16_sw(a.G16, a.max_M, a.N, a.ldg);
  p.dM = a.d_M;
  p.N = a.N;
  p.BN = a.N;
  const int64_t nchunks = ceil_div(ceil_div(std::max<int64_t>(a.max_M, 1), DW16_KR), DW16_CHUNK);
  // at least kmin k-blocks per CTA: each CTA ends with one flush of its
  // whole TMEM sums (2 x 128 x N atomics), which a small M cannot amortise
  const int64_t kmin = std::max(1, env_int("GNNV_DW16_MINKB", 16));
  const int64_t nkbm_ub = ceil_div(std::max<int64_t>(a.max_M, 1), DW16_KR);
  const int splits = (int)std::max<int64_t>(
      1, std::min<int64_t>(std::min<int64_t>(nchunks, (int64_t)(num_sms() / groups)), (int64_t)ceil_div(nkbm_ub, kmin)));
  for (int g = 0; g < groups; ++g) p.sched[g] = sched_slot();
  p.dW = a.dW;
  p.db = a.db;
  // every CTA stores its slice, k_dw16_reduce sums them (no atomics; dW and
  // db are overwritten, so `zeroed` does not matter)
  p.prow = rows + 1;
  p.part = (float*)g_dwpart.get((size_t)splits * p.prow * a.N * sizeof(float), s);
  const size_t bytes = (size_t)DW16_STAGES * (4 + a.N / 64) * DW16_BOX + 8 * (2 * DW16_STAGES + 1) + 4 * DW16_STAGES + 16 + 1024;
  static size_t attr = 0;
  if (bytes > attr) {
    GNNV_TRY_CUDA(cudaFuncSetAttribute(k_tma_dw16, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    attr = bytes;
  }
  const float* dbp = a.dbp;
  int ndbp = a.ndbp;
  const int conv_blocks = 2 * num_sms();
  if (a.G32) {  // G -> bf16 copy + db partials
    float* dbw = (float*)g_dbpart.get((size_t)conv_blocks * a.N * sizeof(float), s);
    launch_k(k_g16_colsum, conv_blocks, 256, 0, s, a.G32, a.ldg32, a.d_M, a.N,
             static_cast<__nv_bfloat16*>(const_cast<void*>(a.G16)), a.ldg, dbw);
    dbp = dbw;
    ndbp = conv_blocks;
    GNNV_CHECK_LAUNCH();
  }
  launch_k(k_tma_dw16, dim3((unsigned)splits, (unsigned)groups), NTHREADS, bytes, s, p);
  GNNV_CHECK_LAUNCH();
  const int64_t total4 = (int64_t)p.prow * (a.N / 4);
  launch_k(k_dw16_reduce, (int)std::min<int64_t>(ceil_div(total4, 32), (int64_t)num_sms() * 8), 256, 0, s, p.part,
           splits, p.prow, a.N, (has_db || dbp) ? 1 : 0, a.dW, a.db, dbp, dbp ? ndbp : 0);
  GNNV_CHECK_LAUNCH();
}

bool gemm_dw_tma(const GemmDwArgs& a, cudaStream_t s) {
  using namespace tma;
  const int BN = rup(a.N, 32);
  if (BN * DW_MT > 512) return false;
  const int nkb1 = (a.K1 + 127) / 128 * 4;  // 32-col blocks per source, whole 128-col tiles
  const int ablocks = a.X2 ? 2 * nkb1 : nkb1;
  const int rows_p = rup(ablocks * 32, BM * DW_MT);
  const int igroups = rows_p / (BM * DW_MT);
  const int64_t nkbm = ceil_div(std::max<int64_t>(a.max_M, 1), DW_KR);
  // >= 8 k-blocks (128 graph rows) per split: small layers use fewer CTAs
  // rather than many short ones whose atomic flush dominates
  const int splits =
      (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(nkbm, 8), (int64_t)num_sms() / igroups));
  const int Ktot = a.X2 ? 2 * a.K1 : a.K1;
  if (!a.zeroed) GNNV_TRY_CUDA(cudaMemsetAsync(a.dW, 0, (size_t)Ktot * a.N * sizeof(float), s));
  Params p{};
  if (a.mask_bits) {
    GNNV_REQUIRE(a.mask_ld == mask_words(a.N), GNNV_ERR_PARAM, "dW: mask bits row stride");
    p.mask = 1;
    p.nwp = a.mask_ld;
    p.th = make_map(reinterpret_cast<const float*>(a.mask_bits), a.max_M, a.mask_ld, a.mask_ld, DW_KR, a.mask_ld,
                    false);
  } else if (a.db_fused) {
    p.dbsum = 1;
  }
  if (p.mask || p.dbsum) {
    GNNV_REQUIRE(a.db, GNNV_ERR_PARAM, "dW: db output required");
    if (!a.zeroed) GNNV_TRY_CUDA(cudaMemsetAsync(a.db, 0, (size_t)a.N * sizeof(float), s));
    p.db = a.db;
  }
  p.x1_rows = a.x1_rows;
  p.ta1 = a.x1_rows ? make_map(a.X1, a.x1_table_rows, a.K1, a.ld1, 1, BM, false)
                    : make_map(a.X1, a.max_M, a.K1, a.ld1, DW_KR, BM, false);
  p.ta2 = a.X2 ? make_map(a.X2, a.max_M, a.K1, a.ld2, DW_KR, BM, false) : p.ta1;
  if (a.G16) {
    GNNV_REQUIRE(a.ldg % 8 == 0, GNNV_ERR_PARAM, "dW: bf16 G row stride must be a multiple of 8");
    p.g16 = 1;
    p.tb = make_map16(a.G16, a.max_M, a.N, a.ldg, DW_KR, BN);
  } else {
    p.tb = make_map(a.G, a.max_M, a.N, a.ldg, DW_KR, BN, false);
  }
  p.two = a.X2 ? 1 : 0;
  p.nkb1 = nkb1;
  p.BN = BN;
  p.dM = a.d_M;
  p.dW = a.dW;
  p.K1 = a.K1;
  p.N = a.N;
  p.splits = splits;
  p.ablocks = ablocks;
  launch<MODE_DW>(p, dim3((unsigned)splits, (unsigned)igroups), s);
  return true;
}

}  // namespace gnnv
