// Node-wise fanout sampling + deterministic first-appearance relabelling.
//
// Paper: Eq.2 unified node-wise sampler; Algorithm 1 line 2
// (P:104-105).  Readings Q1-Q6: exact-k without replacement,
// Philox4x32-10 keyed by (rng_seed; hop, node, draw), Floyd's algorithm,
// ascending CSR position, union frontiers, first-appearance local ids.
//
// Per hop h (all sizes stay on the device; no host round trip):
//   k_sample_hop<G> : one G-lane group per frontier row (G = pow2 >= k).
//                     Lane s computes draw s; Floyd's sequential membership
//                     test is a ballot over the lanes < s; a rank-sort puts
//                     positions in ascending order.  Sampled global ids go to
//                     a fixed-stride slot array ell[r*k + i]; each id not yet
//                     in F_h is "claimed" with atomicMax(tag[u], -(2+slot)),
//                     i.e. the smallest (row, position) slot wins -- exactly
//                     the first appearance in the (dst, position) scan.  The
//                     atomic is skipped when a read already shows an earlier
//                     claim (hub vertices draw thousands of claimants; the
//                     max is monotone, so a stale read only costs an atomic).
//   k_sample_hop_tpr: the same for k <= 8 with one thread per row (more rows
//                     in flight per warp); bit-identical.
//   k_winners       : slot-parallel over the hop: slot e won iff tag[u] still
//                     holds -(2+e); winners collected as per-row bit masks
//                     own[r] (kept: the backward's owner-edge masks).
//   k_relabel_scan  : one thread per row; a single-pass chained scan
//                     (decoupled look-back) over (new ids, sampled count)
//                     gives each row its first new local id and its CSR
//                     offset; winners write tag[u] = n_h + offset + rank and
//                     F[n_h + offset + rank] = u (slot-parallel).
//   k_map           : indices[indptr[r] + i] = tag[ell[r*k+i]] (before the
//                     next hop reuses the slot array, and after the last hop).
//   k_reset         : tag[F_L[i]] = INT_MIN, ready for the next call.
#include <limits.h>

#include <cub/device/device_scan.cuh>

#include "common.cuh"

namespace gnnv {

size_t csc_scan_tmp_bytes(int64_t max_items) {
  size_t bytes = 0;
  GNNV_TRY_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, (const int32_t*)nullptr, (int32_t*)nullptr,
                                              (int)max_items));
  return bytes;
}

constexpr int kScanTile = 256;

__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k.x += 0x9E3779B9u;
      k.y += 0xBB67AE85u;
    }
    const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
  }
  return c;
}

// draw(seed, h, v, s) = word s&3 of Philox(ctr=(s>>2, 0, v, h), key=(lo, hi))
__device__ __forceinline__ uint32_t philox_draw(uint64_t seed, uint32_t h, uint32_t v, uint32_t s) {
  const uint4 o = philox4x32_10(make_uint4(s >> 2, 0u, v, h), make_uint2((uint32_t)seed, (uint32_t)(seed >> 32)));
  const uint32_t w = s & 3u;
  return w == 0 ? o.x : (w == 1 ? o.y : (w == 2 ? o.z : o.w));
}

// One CTA (seeds <= max_seeds, a few thousand): it first clears this
// handle's error flag -- so every sample reports only its own seeds, and a
// bad batch does not poison later steps -- then validates and places the
// seeds.  A seed outside [0, N) is replaced by vertex 0 in F (bit 1 of the
// flag), a repeated seed sets bit 2: every later kernel then indexes only
// valid vertices, and the step reports GNNV_ERR_PARAM at its next sync point
// (its SGD skips the update).
__global__ void __launch_bounds__(1024) k_init_seeds(const int32_t* __restrict__ seeds, int32_t n_seeds, int64_t N,
                                                     int32_t* tag, int32_t* F, int32_t* sizes, int32_t err_index) {
  GNNV_PDL_ENTRY();
  if (threadIdx.x == 0) {
    sizes[err_index] = 0;
    sizes[0] = n_seeds;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n_seeds; i += blockDim.x) {
    const int32_t v = seeds[i];
    if ((uint32_t)v >= (uint64_t)N) {
      F[i] = 0;
      atomicOr(&sizes[err_index], 1);
      continue;
    }
    F[i] = v;
    if (atomicCAS(&tag[v], INT_MIN, i) != INT_MIN) atomicOr(&sizes[err_index], 2);
  }
}

// Four consecutive slots per thread: one 16-byte load of their sampled ids,
// then four independent tag lookups in flight (the slot passes are chains of
// dependent random loads; more of them per thread means fewer waves).
__device__ __forceinline__ void load4(const int32_t* __restrict__ a, int64_t e0, int64_t n, int* v) {
  if (e0 + 3 < n) {
    const int4 q = __ldg(reinterpret_cast<const int4*>(a + e0));
    v[0] = q.x;
    v[1] = q.y;
    v[2] = q.z;
    v[3] = q.w;
  } else {
#pragma unroll
    for (int j = 0; j < 4; ++j) v[j] = e0 + j < n ? __ldg(a + e0 + j) : -1;
  }
}

// Map slots of hop hp (rows [0, n_hp)) to local ids.  Flattened over slots.
__device__ __forceinline__ void map_slots(int64_t t0, int64_t stride, int hp, int kp, const int32_t* sizes,
                                          const int32_t* __restrict__ ellp, const int32_t* __restrict__ cntp,
                                          const int32_t* __restrict__ indptrp, const int32_t* tag,
                                          int32_t* __restrict__ indicesp, int32_t* __restrict__ csc_cnt = nullptr,
                                          uint32_t* __restrict__ lastv = nullptr,
                                          const uint32_t* __restrict__ csc_skip_own = nullptr,
                                          const int32_t* __restrict__ rows_of = nullptr) {
  const int64_t nslots = (int64_t)sizes[hp] * kp;
  for (int64_t e0 = 4 * t0; e0 < nslots; e0 += 4 * stride) {
    int u[4], t[4], dst[4];
    bool owner[4];
    load4(ellp, e0, nslots, u);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t e = e0 + j;
      dst[j] = -1;
      t[j] = 0;
      owner[j] = false;
      if (e < nslots) {
        const int r = (int)(e / kp), i = (int)(e - (int64_t)r * kp);
        if (i < __ldg(cntp + r)) {
          dst[j] = __ldg(indptrp + r) + i;
          t[j] = rows_of ? __ldg(rows_of + u[j]) : tag[u[j]];  // rows_of: the id's cache-table row
          if (csc_skip_own) owner[j] = (__ldg(csc_skip_own + r) >> i) & 1u;
        }
      }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (dst[j] >= 0) {
        indicesp[dst[j]] = t[j];
        if (csc_cnt && !owner[j]) atomicAdd(csc_cnt + t[j], 1);
        if (lastv) atomicMax(lastv + t[j], (uint32_t)dst[j] + 1u);  // the src id's last visit (CSR order)
      }
  }
}

template <int G>
__global__ void __launch_bounds__(256) k_sample_hop(const int64_t* __restrict__ indptr,
                                                    const int32_t* __restrict__ indices, int64_t N,
                                                    const int32_t* __restrict__ F, const int32_t* sizes, int h, int k,
                                                    uint64_t seed, int32_t* __restrict__ ell,
                                                    int32_t* __restrict__ cnt, int32_t* tag, uint32_t* own) {
  GNNV_PDL_ENTRY();
  const int n = sizes[h];
  constexpr int RPW = 32 / G;
  const int lane = threadIdx.x & 31, grp = lane / G, gl = lane % G;
  const unsigned gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (grp * G));
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int base = warp * RPW; base < n; base += nwarps * RPW) {
    const int r = base + grp;
    const bool active = r < n;
    int64_t beg = 0;
    int d = 0, v = 0;
    if (active) {
      v = F[r];
      if ((uint32_t)v < (uint64_t)N) {
        beg = indptr[v];
        d = (int)(indptr[v + 1] - beg);
      }
    }
    const int c = min(k, d);
    int pos = gl, slot = gl;
    if (d > k) {  // group-uniform branch: Floyd's algorithm over k draws
      const int j = d - k + gl;
      uint32_t t = 0;
      if (gl < k) {
        const uint32_t u = philox_draw(seed, (uint32_t)h, (uint32_t)v, (uint32_t)gl);
        t = (uint32_t)(((uint64_t)u * (uint64_t)(uint32_t)(j + 1)) >> 32);
      }
      int sel = (int)t;
      for (int s = 0; s < k; ++s) {
        const int ts = __shfl_sync(gmask, (int)t, s, G);
        const unsigned hit = __ballot_sync(gmask, gl < s && sel == ts);
        if (gl == s && (hit & gmask)) sel = j;
      }
      int rank = 0;
      for (int q = 0; q < k; ++q) {
        const int sq = __shfl_sync(gmask, sel, q, G);
        rank += (sq < sel);
      }
      pos = sel;
      slot = rank;
    }
    if (active && gl < c) {
      const int u = __ldg(&indices[beg + pos]);
      const int e = r * k + slot;
      ell[e] = u;
      if ((uint32_t)u < (uint64_t)N) {
        if (tag && tag[u] < -(2 + e)) atomicMax(&tag[u], -(2 + e));  // skip if an earlier slot already claimed u
      }
    }
    if (active && gl == 0) {
      cnt[r] = c;
      own[r] = 0u;
    }
  }
}

// Thread-per-row variant for small fanouts (k <= KMAX): the same draws and
// the same Floyd recurrence as k_sample_hop, evaluated sequentially by one
// thread per frontier row (4 draws per Philox call), so a warp keeps 32
// independent rows' dependent loads (F -> indptr -> indices -> tag) in
// flight instead of 32/G.  Bit-identical output.
template <int KMAX>
__global__ void __launch_bounds__(256) k_sample_hop_tpr(const int64_t* __restrict__ indptr,
                                                        const int32_t* __restrict__ indices, int64_t N,
                                                        const int32_t* __restrict__ F, const int32_t* sizes, int h,
                                                        int k, uint64_t seed, int32_t* __restrict__ ell,
                                                        int32_t* __restrict__ cnt, int32_t* tag, uint32_t* own) {
  GNNV_PDL_ENTRY();
  const int n = sizes[h];
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
  const int v = F[r];
  int64_t beg = 0;
  int d = 0;
  if ((uint32_t)v < (uint64_t)N) {
    beg = indptr[v];
    d = (int)(indptr[v + 1] - beg);
  }
  const int c = min(k, d);
  int pos[KMAX];
#pragma unroll
  for (int i = 0; i < KMAX; ++i) pos[i] = i;
  if (d > k) {
    const uint2 key = make_uint2((uint32_t)seed, (uint32_t)(seed >> 32));
    uint4 o = make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
    for (int s = 0; s < KMAX; ++s) {
      if (s < k) {
        if ((s & 3) == 0) o = philox4x32_10(make_uint4((uint32_t)s >> 2, 0u, (uint32_t)v, (uint32_t)h), key);
        const uint32_t u = (s & 3) == 0 ? o.x : ((s & 3) == 1 ? o.y : ((s & 3) == 2 ? o.z : o.w));
        const int j = d - k + s;
        const int t = (int)(((uint64_t)u * (uint64_t)(uint32_t)(j + 1)) >> 32);
        bool hit = false;
#pragma unroll
        for (int q = 0; q < KMAX; ++q)
          if (q < s) hit |= pos[q] == t;
        pos[s] = hit ? j : t;
      } else {
        pos[s] = INT_MAX;
      }
    }
    // ascending positions (odd-even transposition network on registers)
#pragma unroll
    for (int pass = 0; pass < KMAX; ++pass) {
#pragma unroll
      for (int q = pass & 1; q + 1 < KMAX; q += 2) {
        const int a = pos[q], b = pos[q + 1];
        pos[q] = min(a, b);
        pos[q + 1] = max(a, b);
      }
    }
  }
  int u[KMAX];
#pragma unroll
  for (int i = 0; i < KMAX; ++i) u[i] = i < c ? __ldg(&indices[beg + pos[i]]) : 0;
#pragma unroll
  for (int i = 0; i < KMAX; ++i) {
    if (i < c) {
      const int e = r * k + i;
      ell[e] = u[i];
      if (tag && (uint32_t)u[i] < (uint64_t)N && tag[u[i]] < -(2 + e)) atomicMax(&tag[u[i]], -(2 + e));
    }
  }
  cnt[r] = c;
  own[r] = 0u;
  }
}

// Winners of hop h's claims, slot-parallel over the whole hop: slot e of
// row r won iff tag[u] still holds its claim code -(2+e) (the smallest slot
// claiming u).  own[r] |= bit i; own[r] was zeroed by the sample kernel.
// The mask doubles as the backward's owner-edge mask (bit i = edge
// indptr[r]+i discovered its src id).
__global__ void k_winners(int64_t N, int h, int k, const int32_t* sizes, const int32_t* __restrict__ ell,
                          const int32_t* __restrict__ cnt, const int32_t* tag, uint32_t* own) {
  GNNV_PDL_ENTRY();
  const int64_t nslots = (int64_t)sizes[h] * k;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e0 = 4 * (blockIdx.x * (int64_t)blockDim.x + threadIdx.x); e0 < nslots; e0 += 4 * stride) {
    int u[4], t[4], r[4], i[4];
    bool ok[4];
    load4(ell, e0, nslots, u);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t e = e0 + j;
      r[j] = (int)(e / k);
      i[j] = (int)(e - (int64_t)r[j] * k);
      ok[j] = e < nslots && i[j] < __ldg(cnt + r[j]) && (uint32_t)u[j] < (uint64_t)N;
      t[j] = ok[j] ? tag[u[j]] : 0;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (ok[j] && t[j] == -(2 + (int)(e0 + j))) atomicOr(&own[r[j]], 1u << i[j]);
  }
}

// NEXT-2: locality-biased node-wise sampling (reading Q26).  One warp per
// frontier row.  Cached neighbours (slot[u] >= 0) weigh W, the others 1;
// the k picks are successive weighted draws without replacement made in
// RANK space (class, rank within the class in ascending CSR position) from
// the same Philox draws as the unbiased sampler: at draw s the remaining
// weight is T = W c + m and t = floor(u_s T / 2^32) selects the (t div W)-th
// remaining cached or the (t - W c)-th remaining uncached neighbour.  Two
// warp sweeps over the adjacency (ballots of the cached flags) count c and
// map the picked ranks to positions (__fns = n-th set bit); positions are
// then sorted ascending.  Bit-identical to oracle.sampler.successive_positions.
__global__ void __launch_bounds__(256) k_sample_hop_biased(const int64_t* __restrict__ indptr,
                                                           const int32_t* __restrict__ indices, int64_t N,
                                                           const int32_t* __restrict__ F, const int32_t* sizes, int h,
                                                           int k, uint64_t seed, const int32_t* __restrict__ slot,
                                                           int W, int32_t* __restrict__ ell, int32_t* __restrict__ cnt,
                                                           int32_t* tag, uint32_t* own) {
  GNNV_PDL_ENTRY();
  __shared__ int s_tc[8][32], s_tu[8][32], s_pos[8][32];
  __shared__ uint32_t s_draw[8][32];
  __shared__ int s_n[8][2];
  const int n = sizes[h];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  int* tc = s_tc[wib];
  int* tu = s_tu[wib];
  int* spos = s_pos[wib];
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int r = warp; r < n; r += nwarps) {
    const int v = F[r];
    int64_t beg = 0;
    int d = 0;
    if ((uint32_t)v < (uint64_t)N) {
      beg = indptr[v];
      d = (int)(indptr[v + 1] - beg);
    }
    const int c = min(k, d);
    int pos = lane;
    if (d > k) {
      int cc = 0;
      for (int p0 = 0; p0 < d; p0 += 32) {
        const int p = p0 + lane;
        const bool f = p < d && __ldg(slot + __ldg(indices + beg + p)) >= 0;
        cc += __popc(__ballot_sync(0xffffffffu, f));
      }
      const int mm = d - cc;
      if (lane < k) s_draw[wib][lane] = philox_draw(seed, (uint32_t)h, (uint32_t)v, (uint32_t)lane);
      __syncwarp();
      if (lane == 0) {
        int nC = 0, nU = 0;
        for (int s = 0; s < k; ++s) {
          const uint32_t crem = (uint32_t)(cc - nC), urem = (uint32_t)(mm - nU);
          const uint32_t T = (uint32_t)W * crem + urem;
          const uint32_t t = (uint32_t)(((uint64_t)s_draw[wib][s] * T) >> 32);
          const bool isc = t < (uint32_t)W * crem;
          int* tk = isc ? tc : tu;
          const int nt = isc ? nC : nU;
          int rnk = (int)(isc ? t / (uint32_t)W : t - (uint32_t)W * crem);
          int ins = 0;
          while (ins < nt && tk[ins] <= rnk) {  // the j-th rank not yet taken
            ++rnk;
            ++ins;
          }
          for (int q = nt; q > ins; --q) tk[q] = tk[q - 1];
          tk[ins] = rnk;
          if (isc) ++nC;
          else ++nU;
        }
        s_n[wib][0] = nC;
        s_n[wib][1] = nU;
      }
      __syncwarp();
      const int nC = s_n[wib][0], nU = s_n[wib][1];
      int iC = 0, iU = 0, cb = 0, ub = 0;
      for (int p0 = 0; p0 < d && (iC < nC || iU < nU); p0 += 32) {
        const int p = p0 + lane;
        const bool valid = p < d;
        const bool f = valid && __ldg(slot + __ldg(indices + beg + p)) >= 0;
        const unsigned bc = __ballot_sync(0xffffffffu, f), bu = __ballot_sync(0xffffffffu, valid && !f);
        const int nc = __popc(bc), nu = __popc(bu);
        while (iC < nC && tc[iC] < cb + nc) {
          const int ln = (int)__fns(bc, 0, tc[iC] - cb + 1);
          if (lane == 0) spos[iC] = p0 + ln;
          ++iC;
        }
        while (iU < nU && tu[iU] < ub + nu) {
          const int ln = (int)__fns(bu, 0, tu[iU] - ub + 1);
          if (lane == 0) spos[nC + iU] = p0 + ln;
          ++iU;
        }
        cb += nc;
        ub += nu;
      }
      __syncwarp();
      // ascending positions: rank of this lane's position among the k
      const int mine = lane < k ? spos[lane] : INT_MAX;
      int rank = 0;
      for (int q = 0; q < k; ++q) rank += spos[q] < mine;
      __syncwarp();
      if (lane < k) spos[rank] = mine;
      __syncwarp();
      pos = lane < k ? spos[lane] : 0;
      __syncwarp();
    }
    if (lane < c) {
      const int u = __ldg(&indices[beg + pos]);
      const int e = r * k + lane;
      ell[e] = u;
      if (tag && (uint32_t)u < (uint64_t)N && tag[u] < -(2 + e)) atomicMax(&tag[u], -(2 + e));
    }
    if (lane == 0) {
      cnt[r] = c;
      own[r] = 0u;
    }
  }
}

__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

constexpr unsigned long long kFlagAgg = 1ull << 62;
constexpr unsigned long long kFlagPre = 2ull << 62;
__device__ __forceinline__ unsigned long long pack2(uint32_t a, uint32_t b) {
  return (unsigned long long)a | ((unsigned long long)b << 31);
}
__device__ __forceinline__ uint32_t unpack_a(unsigned long long w) { return (uint32_t)(w & 0x7FFFFFFFull); }
__device__ __forceinline__ uint32_t unpack_b(unsigned long long w) { return (uint32_t)((w >> 31) & 0x7FFFFFFFull); }

__global__ void __launch_bounds__(kScanTile) k_relabel_scan(int64_t N, int h, int k, int L,
                                                            const int32_t* __restrict__ ell,
                                                            const int32_t* __restrict__ cnt, int32_t* tag,
                                                            int32_t* __restrict__ F, int32_t* __restrict__ indptr,
                                                            uint32_t* __restrict__ own, int32_t* sizes,
                                                            unsigned long long* status,
                                                            uint32_t* __restrict__ lastv,
                                                            int32_t* __restrict__ owner_row) {
  GNNV_PDL_ENTRY();
  __shared__ int s_tile;
  __shared__ uint32_t s_wa[kScanTile / 32], s_wb[kScanTile / 32];
  __shared__ uint32_t s_pa, s_pb;
  const int n = sizes[h];
  const int ntiles = (n + kScanTile - 1) / kScanTile;
  unsigned int* ticket = reinterpret_cast<unsigned int*>(status);
  // tiles are taken in ticket order (the look-back only waits on earlier
  // tickets), so a capped grid may loop over several tiles
  for (;;) {
  if (threadIdx.x == 0) s_tile = (int)atomicAdd(ticket, 1u);
  __syncthreads();
  const int tile = s_tile;
  if (tile >= ntiles) return;
  unsigned long long* st = status + 1;
  const int r = tile * kScanTile + threadIdx.x;
  // winners of the claim (k_winners) as per-row bit masks
  __shared__ uint32_t s_mask[kScanTile];
  const int r0 = tile * kScanTile;
  const int rows = min(kScanTile, n - r0);
  s_mask[threadIdx.x] = threadIdx.x < rows ? own[r0 + threadIdx.x] : 0u;
  const int c = threadIdx.x < rows ? cnt[r0 + threadIdx.x] : 0;
  __syncthreads();
  const uint32_t mask = s_mask[threadIdx.x];
  // block exclusive scan of (a, b) = (#new ids, #sampled)
  const uint32_t a = __popc(mask), b = (uint32_t)c;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t ia = a, ib = b;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t ta = __shfl_up_sync(0xffffffffu, ia, o), tb = __shfl_up_sync(0xffffffffu, ib, o);
    if (lane >= o) {
      ia += ta;
      ib += tb;
    }
  }
  if (lane == 31) {
    s_wa[wid] = ia;
    s_wb[wid] = ib;
  }
  __syncthreads();
  if (wid == 0) {
    uint32_t wa = lane < kScanTile / 32 ? s_wa[lane] : 0, wb = lane < kScanTile / 32 ? s_wb[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t ta = __shfl_up_sync(0xffffffffu, wa, o), tb = __shfl_up_sync(0xffffffffu, wb, o);
      if (lane >= o) {
        wa += ta;
        wb += tb;
      }
    }
    if (lane < kScanTile / 32) {
      s_wa[lane] = wa;  // inclusive over warps
      s_wb[lane] = wb;
    }
  }
  __syncthreads();
  const uint32_t excl_a = ia - a + (wid ? s_wa[wid - 1] : 0u);
  const uint32_t excl_b = ib - b + (wid ? s_wb[wid - 1] : 0u);
  if (wid == 0) {
    // decoupled look-back, one warp: lane j inspects predecessor tile-1-j
    const uint32_t A = s_wa[kScanTile / 32 - 1], B = s_wb[kScanTile / 32 - 1];
    if (tile == 0) {
      if (lane == 0) {
        st_release_u64(&st[0], kFlagPre | pack2(A, B));
        s_pa = 0;
        s_pb = 0;
      }
    } else {
      if (lane == 0) st_release_u64(&st[tile], kFlagAgg | pack2(A, B));
      uint32_t pa = 0, pb = 0;
      int p = tile - 1;
      while (true) {
        const int q = p - lane;
        unsigned long long w = kFlagPre;  // before tile 0: an inclusive zero
        if (q >= 0) {
          do {
            w = ld_acquire_u64(&st[q]);
          } while ((w >> 62) == 0);
        }
        const unsigned pre = __ballot_sync(0xffffffffu, (w >> 62) == 2);
        const int stop = pre ? __ffs(pre) - 1 : 31;  // nearest inclusive prefix in the window
        uint32_t va = lane <= stop ? unpack_a(w) : 0u, vb = lane <= stop ? unpack_b(w) : 0u;
#pragma unroll
        for (int o = 16; o; o >>= 1) {
          va += __shfl_xor_sync(0xffffffffu, va, o);
          vb += __shfl_xor_sync(0xffffffffu, vb, o);
        }
        pa += va;
        pb += vb;
        if (pre) break;
        p -= 32;
      }
      if (lane == 0) {
        st_release_u64(&st[tile], kFlagPre | pack2(pa + A, pb + B));
        s_pa = pa;
        s_pb = pb;
      }
    }
  }
  __syncthreads();
  const uint32_t new_off = s_pa + excl_a, edge_off = s_pb + excl_b;
  if (r < n) {
    indptr[r] = (int32_t)edge_off;
    if (lastv) lastv[r] = 0u;        // last-use slots of this hop's src ids, set by k_map
    if (owner_row) owner_row[r] = -1;  // the dst prefix has no owner edge in this hop
  }
  __shared__ uint32_t s_off[kScanTile];
  s_off[threadIdx.x] = new_off;
  __syncthreads();
  // winners get their local ids slot-parallel: row offset + rank of the
  // slot among the row's winners (no per-row serial chain)
  {
    const int nslots = rows * k;
    for (int j = threadIdx.x; j < nslots; j += kScanTile) {
      const int rl = j / k, i = j - rl * k;
      const uint32_t m = s_mask[rl];
      if ((m >> i) & 1u) {
        const int u = ell[r0 * k + j];
        const int nid = n + (int)s_off[rl] + __popc(m & ((1u << i) - 1u));
        tag[u] = nid;
        F[nid] = u;
        if (lastv) lastv[nid] = 0u;
        if (owner_row) owner_row[nid] = r0 + rl;  // the dst row whose edge discovered u
      }
    }
  }
  if (tile == ntiles - 1 && threadIdx.x == kScanTile - 1) {
    const uint32_t tot_a = new_off + a, tot_b = edge_off + b;
    sizes[h + 1] = n + (int)tot_a;
    sizes[L + 1 + h] = (int)tot_b;
    indptr[n] = (int32_t)tot_b;
  }
  __syncthreads();  // shared state is reused by the next tile
  }
}

// Also clears the scan status words hop hp's k_relabel_scan used (its
// ticket counter and one word per tile), so the next hop's -- or the next
// batch's -- scan starts from zero without a memset node in the stream.
// With csc_cnt (hops that get a CSC): also counts each src id's in-edges.
__global__ void k_map(int hp, int kp, const int32_t* sizes, const int32_t* __restrict__ ellp,
                      const int32_t* __restrict__ cntp, const int32_t* __restrict__ indptrp, const int32_t* tag,
                      int32_t* __restrict__ indicesp, unsigned long long* scan, int64_t scan_words,
                      int32_t* __restrict__ csc_cnt, uint32_t* __restrict__ lastv,
                      const uint32_t* __restrict__ csc_skip_own, const int32_t* __restrict__ rows_of) {
  GNNV_PDL_ENTRY();
  const int64_t t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t used = std::min<int64_t>(scan_words, 1 + ((int64_t)sizes[hp] + kScanTile - 1) / kScanTile);
  for (int64_t i = t0; i < used; i += stride) scan[i] = 0ull;
  map_slots(t0, stride, hp, kp, sizes, ellp, cntp, indptrp, tag, indicesp, csc_cnt, lastv, csc_skip_own, rows_of);
}

// CSC fill of hop hp (counting sort): colptr = exclusive scan of the in-edge
// counts; edge (r, u) takes slot colptr[u] + (--cnt[u]), which also leaves
// the counts zeroed for the next batch.  The order of a column's entries
// follows the atomics; the pulled sum is exact up to that order.
// csc_skip_own != NULL: the owner edges (bit i of own[r]) are left out --
// the fused L2 push handles them as runs (owner rows).
__global__ void k_csc_fill(int hp, int kp, const int32_t* sizes, const int32_t* __restrict__ indptrp,
                           const int32_t* __restrict__ indicesp, int32_t* __restrict__ csc_cnt,
                           const int32_t* __restrict__ colptr, int32_t* __restrict__ csc,
                           const uint32_t* __restrict__ csc_skip_own) {
  GNNV_PDL_ENTRY();
  const int64_t nslots = (int64_t)sizes[hp] * kp;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nslots; e += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(e / kp), i = (int)(e - (int64_t)r * kp);
    const int beg = __ldg(indptrp + r);
    if (csc_skip_own && ((__ldg(csc_skip_own + r) >> i) & 1u)) continue;
    if (i < __ldg(indptrp + r + 1) - beg) {
      const int u = __ldg(indicesp + beg + i);
      csc[__ldg(colptr + u) + atomicSub(csc_cnt + u, 1) - 1] = r;
    }
  }
}

// Tags of F_L back to empty.  With rowidx (whole-table trainer): also every
// F_L row's cache row, rowidx[i] = slot[F[i]], and the gather counters of
// a cache that holds every row (n_L local hits) -- the trainer then needs
// no gather pass.
// the last hop kept as table rows: F_L = F_{L-1}; its edge count and the
// CSR's closing offset from the exclusive sum of the row counts
__global__ void k_last_hop_sizes(int32_t* sizes, int L, int32_t* indptr, const int32_t* cnt) {
  GNNV_PDL_ENTRY();
  if (threadIdx.x == 0) {
    const int n = sizes[L - 1];
    const int e = n ? indptr[n - 1] + cnt[n - 1] : 0;
    indptr[n] = e;
    sizes[L] = n;
    sizes[L + 1 + (L - 1)] = e;
  }
}

__global__ void k_reset(const int32_t* __restrict__ F, const int32_t* sizes, int L, int64_t N, int32_t* tag,
                        const int32_t* __restrict__ slot, int32_t* __restrict__ rowidx,
                        unsigned long long* __restrict__ stats) {
  GNNV_PDL_ENTRY();
  const int64_t n = sizes[L];
  if (stats && blockIdx.x == 0 && threadIdx.x == 0) {
    stats[0] = (unsigned long long)n;
    stats[1] = (unsigned long long)n;
    stats[2] = 0ull;
    stats[3] = 0ull;
  }
  for (int64_t i0 = 4 * (blockIdx.x * (int64_t)blockDim.x + threadIdx.x); i0 < n;
       i0 += 4 * (int64_t)gridDim.x * blockDim.x) {
    int v[4];
    load4(F, i0, n, v);
    int r[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) r[j] = (rowidx && (uint32_t)v[j] < (uint64_t)N) ? __ldg(slot + v[j]) : 0;
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if ((uint32_t)v[j] < (uint64_t)N) tag[v[j]] = INT_MIN;
    if (rowidx) {
      if (i0 + 3 < n) {
        *reinterpret_cast<int4*>(rowidx + i0) = make_int4(r[0], r[1], r[2], r[3]);
      } else {
        for (int j = 0; j < 4 && i0 + j < n; ++j) rowidx[i0 + j] = r[j];
      }
    }
  }
}

// One work item per thread / row group (no grid-stride loops over a capped
// grid): short-lived blocks let the step's higher-priority kernels
// interleave with a prefetch.  Grids are sized by the Eq.12 capacity of the
// hop (the realised size is on the device); surplus blocks exit at once.
static int grid_for(int64_t work, int per_block) { return capped_grid(ceil_div(std::max<int64_t>(work, 1), per_block)); }

void launch_sample(gnnv_graph* g, gnnv_blocks* b, const int32_t* d_seeds, int32_t n_seeds, uint64_t rng_seed,
                   cudaStream_t s) {
  const int L = b->L;
  const int err_index = 2 * L + 1;
  launch_k(k_init_seeds, 1, 1024, 0, s, d_seeds, n_seeds, g->n, b->d_tag, b->d_F, b->d_sizes, err_index);
  GNNV_CHECK_LAUNCH();
  // Hop h's slots reuse d_ell / d_cnt, so hop h-1 is mapped to local ids
  // (its tags are final after its scan) before hop h samples.  Hops with a
  // CSC (bit hp of csc_mask) then sort their edges by src id (stable: dst order
  // within a column) and derive the column pointers.
  auto map_hop = [&](int hp) {
    const int64_t slots_ub = b->max_nnz[hp];
    const bool csc = (b->csc_mask >> hp) & 1u;
    launch_k(k_map, grid_for(slots_ub, 1024), 256, 0, s, hp, b->fanouts[hp], b->d_sizes, b->d_ell, b->d_cnt,
             b->d_indptr[hp], b->d_tag, b->d_indices[hp], b->d_scan, b->scan_words,
             csc ? b->d_csc_cnt : (int32_t*)nullptr, hp == L - 1 ? b->d_lastv : (uint32_t*)nullptr,
             csc && ((b->csc_nonowner >> hp) & 1u) ? b->d_own[hp] : (const uint32_t*)nullptr,
             hp == L - 1 ? b->last_rows : (const int32_t*)nullptr);
    GNNV_CHECK_LAUNCH();
    if (!csc) return;
    size_t tmp = b->csc_tmp_bytes;
    GNNV_TRY_CUDA(cub::DeviceScan::ExclusiveSum(b->d_csc_tmp, tmp, b->d_csc_cnt, b->d_colptr[hp],
                                                (int)(b->max_n[hp + 1] + 1), s));
    GNNV_CHECK_LAUNCH();
    launch_k(k_csc_fill, grid_for(slots_ub, 256), 256, 0, s, hp, b->fanouts[hp], b->d_sizes, b->d_indptr[hp],
             b->d_indices[hp], b->d_csc_cnt, b->d_colptr[hp], b->d_csc[hp],
             ((b->csc_nonowner >> hp) & 1u) ? b->d_own[hp] : (const uint32_t*)nullptr);
    GNNV_CHECK_LAUNCH();
  };
  for (int h = 0; h < L; ++h) {
    const int k = b->fanouts[h];
    const int64_t rows_ub = b->max_n[h];
    if (h > 0) map_hop(h - 1);
    const int threads = 256;
    // the whole-table trainer's last hop (b->last_rows): no claims, no local ids
    int32_t* const tagh = (h == L - 1 && b->last_rows) ? nullptr : b->d_tag;
#define GNNV_SAMPLE_LAUNCH(G)                                                                              \
  launch_k(k_sample_hop<G>, grid_for(rows_ub, threads / 32 * (32 / G)), threads, 0, s,                  \
      g->d_indptr, g->d_indices, g->n, b->d_F, b->d_sizes, h, k, rng_seed, b->d_ell, b->d_cnt, tagh, b->d_own[h])
    if (b->loc_w > 1) {
      launch_k(k_sample_hop_biased, grid_for(rows_ub, 8), 256, 0, s, g->d_indptr, g->d_indices, g->n, b->d_F,
               b->d_sizes, h, k, rng_seed, b->loc_slot, (int)b->loc_w, b->d_ell, b->d_cnt, tagh, b->d_own[h]);
    } else if (k <= 4) {
      launch_k(k_sample_hop_tpr<4>, grid_for(rows_ub, threads), threads, 0, s, 
          g->d_indptr, g->d_indices, g->n, b->d_F, b->d_sizes, h, k, rng_seed, b->d_ell, b->d_cnt, tagh, b->d_own[h]);
    } else if (k <= 8) {
      launch_k(k_sample_hop_tpr<8>, grid_for(rows_ub, threads), threads, 0, s, 
          g->d_indptr, g->d_indices, g->n, b->d_F, b->d_sizes, h, k, rng_seed, b->d_ell, b->d_cnt, tagh, b->d_own[h]);
    } else if (k <= 16 && rows_ub < 16384) {
      GNNV_SAMPLE_LAUNCH(16);  // few rows: lanes per row beat rows per thread
    } else if (k <= 16) {
      launch_k(k_sample_hop_tpr<16>, grid_for(rows_ub, threads), threads, 0, s, 
          g->d_indptr, g->d_indices, g->n, b->d_F, b->d_sizes, h, k, rng_seed, b->d_ell, b->d_cnt, tagh, b->d_own[h]);
    } else {
      GNNV_SAMPLE_LAUNCH(32);
    }
#undef GNNV_SAMPLE_LAUNCH
    GNNV_CHECK_LAUNCH();
    const int tiles_ub = capped_grid(ceil_div(rows_ub, kScanTile));
    if (tagh) {  // no winners without claims: own[] stays zero, the scan numbers no new ids
      launch_k(k_winners, grid_for(rows_ub * k, 1024), 256, 0, s, g->n, h, k, b->d_sizes, b->d_ell, b->d_cnt, b->d_tag,
               b->d_own[h]);
      GNNV_CHECK_LAUNCH();
    }
    if (!tagh) {
      // the last hop as table rows numbers no new ids: its CSR offsets are a
      // plain exclusive sum of the row counts (cub, over the row capacity;
      // entries past the hop's n are never read), the totals fixed up after
      size_t tmp = b->csc_tmp_bytes;
      GNNV_TRY_CUDA(cub::DeviceScan::ExclusiveSum(b->d_csc_tmp, tmp, b->d_cnt, b->d_indptr[h], (int)rows_ub, s));
      GNNV_CHECK_LAUNCH();
      launch_k(k_last_hop_sizes, 1, 32, 0, s, b->d_sizes, L, b->d_indptr[h], b->d_cnt);
      GNNV_CHECK_LAUNCH();
      continue;
    }
    launch_k(k_relabel_scan, tiles_ub, kScanTile, 0, s, g->n, h, k, L, b->d_ell, b->d_cnt, b->d_tag, b->d_F,
                                                  b->d_indptr[h], b->d_own[h], b->d_sizes, b->d_scan,
             h == L - 1 ? b->d_lastv : (uint32_t*)nullptr, b->d_owner_row[h]);
    GNNV_CHECK_LAUNCH();
  }
  map_hop(L - 1);
  launch_k(k_reset, grid_for(b->max_n[L], 1024), 256, 0, s, b->d_F, b->d_sizes, L, g->n, b->d_tag, b->rowidx_slot,
           b->d_rowidx, reinterpret_cast<unsigned long long*>(b->d_rowidx_stats));
  GNNV_CHECK_LAUNCH();
}

}  // namespace gnnv
