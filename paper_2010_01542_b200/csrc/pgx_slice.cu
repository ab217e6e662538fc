// pgx_slice.cu -- the partitioned (multi-GPU) superstep, one phase per
// launch: scatter into a full-width mailbox, apply on the owned slice.
// The host (paper_2010_01542_b200/distributed.py) reduces the mailbox
// slices onto their owners between the two (NCCL via torch.distributed).
#include "pgx_apply.cuh"
#include "pgx_common.cuh"
#include "pgx_gather.cuh"
#include "pgx_scatter.cuh"
#include "pgx_seg.cuh"

namespace pgx {
namespace {

// ------------------------------------------------------------------
// phase kernels of the partitioned (multi-GPU) superstep, SURVEY 8(e).
// Each rank owns the out-edges of a contiguous vertex range [lo, lo+len)
// and a slice of the mailbox.  Per superstep: K1 scatters the rank's
// senders into a FULL-WIDTH local mailbox (global destination ids); the
// host reduces the mailbox slices onto their owners (NCCL min / sum);
// K2 applies on the owned slice (has-message == mailbox != neutral after
// the min reduction: messages are < n <= 2^31 and never the neutral).
// Regular (non-cooperative) stream-ordered launches.
// ------------------------------------------------------------------

struct SliceCounters {       // device counters of one partitioned superstep
  unsigned long long packed; // senders << 32 | edges of the next frontier
  unsigned long long recip;  // recipients in the owned slice
  unsigned long long bcast;  // vertices that computed a new value
  double dangling;           // PageRank: rank mass of owned dangling vertices
};

#ifndef PGX_SCATTER_MIN_BLOCKS
#define PGX_SCATTER_MIN_BLOCKS PGX_MIN_BLOCKS
#endif

template <int OP, MsgSrc MS, bool PEER = false, bool BFS = false>
__global__ void __launch_bounds__(kBlock, PGX_SCATTER_MIN_BLOCKS) scatter_kernel(ScatterArgs a,
                                                                          int read_filter) {
  extern __shared__ __align__(16) char smem[];
  scatter_phase<OP, MS, 0, PEER, BFS>(a, smem, read_filter != 0);
  // the peer reds are performed at system scope before the kernel ends, so
  // the collective that follows it on the stream orders them before the
  // owners' apply
  if (PEER) __threadfence_system();
}

template <int APP>
__global__ void __launch_bounds__(kBlock) apply_slice_kernel(
    int32_t len, const int32_t *__restrict__ row_ptr, uint32_t *val, uint32_t *mailbox,
    int32_t *f_eb, int32_t *f_rs, uint32_t *f_msg, int32_t *tile_src, SliceCounters *ctr,
    int32_t count_only, uint32_t neutral, uint32_t *sv) {
  __shared__ unsigned long long s_w[33];
  __shared__ unsigned long long s_gbase;
  __shared__ unsigned long long s_red[32];
  constexpr int kI = 4;
  const int base = blockIdx.x * kBlock * kI;
  int deg[kI], rs[kI];
  uint32_t m[kI];
  unsigned long long mine = 0, recips = 0, bcast = 0;
#pragma unroll
  for (int j = 0; j < kI; j++) {
    const int v = base + j * kBlock + threadIdx.x;
    deg[j] = 0;
    m[j] = (v < len) ? mailbox[v] : neutral;
    if (m[j] != neutral) {
      recips++;
      if (!count_only) {
        mailbox[v] = neutral;  // consume
        if (m[j] < val[v]) {
          val[v] = m[j];
          bcast++;
          rs[j] = row_ptr[v];
          deg[j] = row_ptr[v + 1] - rs[j];
          if (deg[j] > 0) mine += (1ull << 32) | (unsigned long long)deg[j];
        }
      }
    }
  }
  unsigned long long total;
  unsigned long long run = block_excl_scan_u64(mine, s_w, &total);
  if (total) {
    if (threadIdx.x == 0) s_gbase = atomicAdd(&ctr->packed, total);
    __syncthreads();
    run += s_gbase;
#pragma unroll
    for (int j = 0; j < kI; j++) {
      if (deg[j] > 0) {
        const unsigned pos = (unsigned)(run >> 32);
        const int eb = (int)(run & 0xFFFFFFFFull);
        f_eb[pos] = eb;
        f_rs[pos] = rs[j];
        f_msg[pos] = (APP == PGX_APP_SSSP) ? m[j] + 1u : m[j];
        if (sv) sv[base + j * kBlock + threadIdx.x] = m[j];  // CC: the label it sends (K1s)
        for (int64_t t = ((int64_t)eb + kTile - 1) / kTile; t * kTile < (int64_t)eb + deg[j]; t++)
          tile_src[t] = (int)pos;
        run += (1ull << 32) | (unsigned long long)deg[j];
      }
    }
  }
  recips = block_sum<unsigned long long>(recips, s_red);
  if (threadIdx.x == 0 && recips) atomicAdd(&ctr->recip, recips);
  bcast = block_sum<unsigned long long>(bcast, s_red);
  if (threadIdx.x == 0 && bcast) atomicAdd(&ctr->bcast, bcast);
}

// PageRank apply of an owned slice.  `dangling` is the job's dangling mass
// after the previous superstep (device scalar: summed over ranks by a
// collective on the stream, no host read), dn = dangling / n as in the
// single-GPU kernel (algorithms.py:61-73).
__global__ void __launch_bounds__(kBlock) pr_apply_slice_kernel(
    int32_t len, const int32_t *__restrict__ row_ptr, double *rank, double *mailbox,
    double *share, double base, double damping, const double *dangling, double n_total,
    int32_t last, double *partials) {
  __shared__ double s_red[32];
  const double dn = __ddiv_rn(*dangling, n_total);
  const int v = blockIdx.x * kBlock + threadIdx.x;
  double my_d = 0.0;
  if (v < len) {
    const double folded = mailbox[v];
    mailbox[v] = 0.0;
    const double r = __dadd_rn(base, __dmul_rn(damping, __dadd_rn(folded, dn)));
    rank[v] = r;
    const int deg = row_ptr[v + 1] - row_ptr[v];
    if (deg == 0) my_d = r;
    else if (!last) share[v] = __ddiv_rn(r, (double)deg);
  }
  const double b = block_sum<double>(my_d, s_red);
  if (threadIdx.x == 0) partials[blockIdx.x] = b;
}

// Pull fold of a rank's slice (the reference's PR mode, engine.py:425-457):
// K3 over the rank's local in-CSR (rows = padded mailbox positions, ids =
// local sources), writing the full-width partial fold; rows spanning tiles
// leave head / tail partials for fold_spanning_kernel.
__global__ void __launch_bounds__(kBlock, PGX_MIN_BLOCKS) gather_slice_kernel(GatherArgs g) {
  extern __shared__ __align__(16) char smem[];
  gather_phase(g, smem);
}

// Unit-weight SSSP apply of the owned block after a bitmap exchange: the
// recipients are the set bits of the rank's block of its has-bitmap (its
// own scatter's and the peers' red.or); an unreached recipient takes
// distance `level` and, with out-edges, joins the next frontier with
// message level + 1.  The block's bits are consumed (cleared).
__global__ void __launch_bounds__(kBlock) apply_slice_bfs_kernel(
    int32_t len, const int32_t *__restrict__ row_ptr, uint32_t *val, uint32_t *has_block,
    int32_t *f_eb, int32_t *f_rs, uint32_t *f_msg, int32_t *tile_src, SliceCounters *ctr,
    int32_t count_only, uint32_t level) {
  __shared__ unsigned long long s_w[33];
  __shared__ unsigned long long s_gbase;
  __shared__ unsigned long long s_red[32];
  constexpr int kI = 4;
  const int base = blockIdx.x * kBlock * kI;
  int deg[kI], rs[kI];
  unsigned long long mine = 0, recips = 0, bcast = 0;
#pragma unroll
  for (int j = 0; j < kI; j++) {
    const int v = base + j * kBlock + threadIdx.x;
    deg[j] = 0;
    const bool got = v < len && ((has_block[v >> 5] >> (v & 31)) & 1u);
    if (got) {
      recips++;
      if (!count_only && val[v] == kNeutralMin) {
        val[v] = level;
        bcast++;
        rs[j] = row_ptr[v];
        deg[j] = row_ptr[v + 1] - rs[j];
        if (deg[j] > 0) mine += (1ull << 32) | (unsigned long long)deg[j];
      }
    }
  }
  unsigned long long total;
  unsigned long long run = block_excl_scan_u64(mine, s_w, &total);
  if (total) {
    if (threadIdx.x == 0) s_gbase = atomicAdd(&ctr->packed, total);
    __syncthreads();
    run += s_gbase;
#pragma unroll
    for (int j = 0; j < kI; j++) {
      if (deg[j] > 0) {
        const unsigned pos = (unsigned)(run >> 32);
        const int eb = (int)(run & 0xFFFFFFFFull);
        f_eb[pos] = eb;
        f_rs[pos] = rs[j];
        f_msg[pos] = level + 1u;
        for (int64_t t = ((int64_t)eb + kTile - 1) / kTile; t * kTile < (int64_t)eb + deg[j]; t++)
          tile_src[t] = (int)pos;
        run += (1ull << 32) | (unsigned long long)deg[j];
      }
    }
  }
  recips = block_sum<unsigned long long>(recips, s_red);
  if (threadIdx.x == 0 && recips) atomicAdd(&ctr->recip, recips);
  bcast = block_sum<unsigned long long>(bcast, s_red);
  if (threadIdx.x == 0 && bcast) atomicAdd(&ctr->bcast, bcast);
}

// the owned block's bits consumed (after every thread read them)
__global__ void clear_words_kernel(uint32_t *w, int32_t count) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < count; i += gridDim.x * blockDim.x)
    w[i] = 0u;
}

// K1s on a rank's slice: the destination-segmented scatter of the rank's
// local CSR (destinations = padded mailbox positions) into its full-width
// mailbox; message = global source id (superstep 0) or the send value.
template <int MSG>
__global__ void __launch_bounds__(kBlock, PGX_MIN_BLOCKS) seg_slice_kernel(SegPass sp) {
  extern __shared__ __align__(16) char smem[];
  seg_scatter_phase<MSG>(sp, smem);
}

// rows whose in-edges span tiles: tail of the first tile + heads of the
// later ones, in tile order (the persistent kernel's combine)
__global__ void fold_spanning_kernel(int32_t nspan, const int32_t *rows, const int32_t *t0,
                                     const int32_t *t1, const double *head, const double *tail,
                                     double *folded) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nspan; i += gridDim.x * blockDim.x) {
    const int a = t0[i], b = t1[i];
    folded[rows[i]] = span_sum(head, tail, a, b);
  }
}

__global__ void slice_init_kernel(int app, int32_t len, int32_t lo, uint32_t *val,
                                  const int32_t *row_ptr, double *rank, double *share,
                                  double r0) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < len; v += gridDim.x * blockDim.x) {
    if (app == PGX_APP_CC) val[v] = (uint32_t)(lo + v);
    else if (app == PGX_APP_SSSP) val[v] = kNeutralMin;
    else {
      const int deg = row_ptr[v + 1] - row_ptr[v];
      rank[v] = r0;
      share[v] = deg ? __ddiv_rn(r0, (double)deg) : 0.0;
    }
  }
}


// ---- sparse exchange -------------------------------
// The touched slots of the full-width local mailbox are its set has-bits.
// Those outside the rank's own range [lo, hi) are counted, or compacted in
// vertex order into (slot << 32 | value) pairs -- which groups them by
// owner -- and reset to the neutral; the owner min-combines the pairs it
// receives into its slice.

__device__ __forceinline__ uint32_t foreign_bits(const uint32_t *has, int wi, int32_t n, int32_t lo,
                                                 int32_t hi) {
  uint32_t w = has[wi];
  const int v0 = wi << 5;
  if (v0 + 32 > n) w &= (n - v0 >= 32) ? 0xFFFFFFFFu : ((1u << (n - v0)) - 1u);
  // drop bits in [lo, hi)
  const int a = max(lo - v0, 0), b = min(hi - v0, 32);
  if (a < b) {
    const uint32_t hi_mask = (b >= 32) ? 0xFFFFFFFFu : ((1u << b) - 1u);
    const uint32_t lo_mask = (1u << a) - 1u;
    w &= ~(hi_mask & ~lo_mask);
  }
  return w;
}

__global__ void __launch_bounds__(kCompactBlock) touched_count_kernel(
    const uint32_t *has, int32_t n, int32_t lo, int32_t hi, int32_t *blk) {
  __shared__ int s_warp[33];
  const int words = (n + 31) >> 5;
  const int wi = blockIdx.x * kCompactBlock + threadIdx.x;
  const int c = (wi < words) ? __popc(foreign_bits(has, wi, n, lo, hi)) : 0;
  int total;
  block_excl_scan(c, s_warp, &total);
  if (threadIdx.x == 0) blk[blockIdx.x] = total;
}

__global__ void __launch_bounds__(kCompactBlock) touched_scan_kernel(int32_t *blk, int32_t nb,
                                                                    int64_t *count) {
  __shared__ int s_warp[33];
  int carry = 0;
  for (int base = 0; base < nb; base += kCompactBlock) {
    const int i = base + threadIdx.x;
    const int x = (i < nb) ? blk[i] : 0;
    int total;
    const int ex = block_excl_scan(x, s_warp, &total);
    if (i < nb) blk[i] = carry + ex;
    carry += total;
  }
  if (threadIdx.x == 0) *count = carry;
}

__global__ void __launch_bounds__(kCompactBlock) touched_write_kernel(
    const uint32_t *has, int32_t n, int32_t lo, int32_t hi, const int32_t *blk, uint32_t *mailbox,
    uint32_t neutral, unsigned long long *pairs) {
  __shared__ int s_warp[33];
  const int words = (n + 31) >> 5;
  const int wi = blockIdx.x * kCompactBlock + threadIdx.x;
  const uint32_t w = (wi < words) ? foreign_bits(has, wi, n, lo, hi) : 0u;
  int total;
  int pos = blk[blockIdx.x] + block_excl_scan(__popc(w), s_warp, &total);
  uint32_t rem = w;
  while (rem) {
    const int b = __ffs(rem) - 1;
    rem &= rem - 1;
    const int v = (wi << 5) + b;
    const uint32_t m = mailbox[v];
    mailbox[v] = neutral;
    pairs[pos++] = ((unsigned long long)(uint32_t)v << 32) | m;
  }
}

// Peer exchange epilogue: the foreign slots this rank touched (its local
// filter copies) go back to the neutral and every has-bit is cleared; the
// owned slots were consumed by the apply.
__global__ void reset_touched_kernel(uint32_t *has, int32_t n, int32_t lo, int32_t hi,
                                     uint32_t *mailbox, uint32_t neutral) {
  const int words = (n + 31) >> 5;
  for (int wi = blockIdx.x * blockDim.x + threadIdx.x; wi < words;
       wi += gridDim.x * blockDim.x) {
    if (!has[wi]) continue;
    uint32_t rem = foreign_bits(has, wi, n, lo, hi);
    // only words with foreign bits (owned ranges are whole words): an owned
    // word may already be receiving the peers' next-superstep bits (the
    // unit-weight SSSP bitmap exchange) and is never written here
    if (!rem) continue;
    has[wi] = 0u;
    while (rem) {
      const int b = __ffs(rem) - 1;
      rem &= rem - 1;
      mailbox[(wi << 5) + b] = neutral;
    }
  }
}

__global__ void scatter_pairs_min_kernel(const unsigned long long *pairs, int64_t count,
                                         uint32_t *mailbox) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long p = pairs[i];
    red_min_u32(mailbox + (uint32_t)(p >> 32), (uint32_t)(p & 0xFFFFFFFFull));
  }
}

}  // namespace
}  // namespace pgx

using namespace pgx;

extern "C" {

int pgx_slice_init(int app, int32_t len, int32_t lo, void *val, const int32_t *row_ptr,
                   double *share, double r0, uintptr_t stream) {
  if (len < 0 || !val || (app == PGX_APP_PAGERANK && (!row_ptr || !share)))
    return fail(PGX_EINVAL, "bad slice_init arguments");
  if (!len) return PGX_OK;
  const int grid = (int)std::min<int64_t>(ceil_div(len, 256), 148 * 16);
  slice_init_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(
      app, len, lo, (uint32_t *)val, row_ptr, (double *)val, share, r0);
  PGX_CUDA(cudaGetLastError());
  return PGX_OK;
}

int pgx_scatter(int op, int dense, const int32_t *col_idx, const int32_t *src_eb,
                const int32_t *src_rs, const int32_t *src_ids, int32_t id_offset,
                const void *src_msg, const int32_t *tile_src, int32_t nsrc, int64_t edges,
                void *mailbox, uint32_t *has_bits, uint32_t neutral, uintptr_t stream) {
  if (op != PGX_OP_MIN_U32 && op != PGX_OP_SUM_F64) return fail(PGX_EINVAL, "unknown op");
  if (edges < 0 || edges > INT32_MAX || nsrc < 0) return fail(PGX_EINVAL, "bad sizes");
  if (edges == 0) return PGX_OK;
  if (!col_idx || !src_eb || !tile_src || !mailbox || (!dense && (!src_rs || !src_msg)) ||
      (dense && !src_ids) || (op == PGX_OP_SUM_F64 && !src_msg))
    return fail(PGX_EINVAL, "null scatter pointer");
  ScatterArgs a;
  a.col = col_idx;
  a.eb = src_eb;
  a.rs = src_rs;
  a.ids = src_ids;
  a.msg = src_msg;
  a.tile_src = tile_src;
  a.nsrc = nsrc;
  a.E = edges;
  a.mailbox = mailbox;
  a.has = has_bits;
  a.id_offset = id_offset;
  a.hub_ids = nullptr;
  a.nhubs = 0;
  a.cas_loop = 0;
  a.neutral = neutral;
  a.n = INT32_MAX;  // the slice ABI has no vertex count: unchecked
  const int64_t tiles = ceil_div(edges, kTile);
  int sms = 148, dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(tiles, kWarps),
                                                               (int64_t)sms * PGX_SCATTER_MIN_BLOCKS));
  cudaStream_t st = (cudaStream_t)stream;
  const size_t smem = scatter_smem(op);
  const int rf = g_opt[PGX_OPT_READ_FILTER];
  if (op == PGX_OP_MIN_U32 && !dense) {
    PGX_CUDA(cudaFuncSetAttribute(scatter_kernel<PGX_OP_MIN_U32, MsgSrc::kFrontier>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    scatter_kernel<PGX_OP_MIN_U32, MsgSrc::kFrontier><<<grid, kBlock, smem, st>>>(a, rf);
  } else if (op == PGX_OP_MIN_U32) {
    PGX_CUDA(cudaFuncSetAttribute(scatter_kernel<PGX_OP_MIN_U32, MsgSrc::kSourceId>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    scatter_kernel<PGX_OP_MIN_U32, MsgSrc::kSourceId><<<grid, kBlock, smem, st>>>(a, rf);
  } else if (dense) {
    PGX_CUDA(cudaFuncSetAttribute(scatter_kernel<PGX_OP_SUM_F64, MsgSrc::kShareById>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    scatter_kernel<PGX_OP_SUM_F64, MsgSrc::kShareById><<<grid, kBlock, smem, st>>>(a, rf);
  } else {
    return fail(PGX_EINVAL, "sum scatter needs the dense sender list");
  }
  PGX_CUDA(cudaGetLastError());
  return PGX_OK;
}

int pgx_scatter_peer(int dense, const int32_t *col_idx, const int32_t *src_eb,
                     const int32_t *src_rs, const int32_t *src_ids, int32_t id_offset,
                     const void *src_msg, const int32_t *tile_src, int32_t nsrc, int64_t edges,
                     uint32_t *mailbox, uint32_t *has_bits, uint32_t neutral,
                     const uint64_t *peer_mailboxes, const int32_t *bounds, int32_t world,
                     int32_t lo, int32_t hi, uintptr_t stream) {
  if (edges < 0 || edges > INT32_MAX || nsrc < 0) return fail(PGX_EINVAL, "bad sizes");
  if (world < 1 || lo < 0 || hi < lo || !peer_mailboxes || !bounds)
    return fail(PGX_EINVAL, "bad peer arguments");
  if (edges == 0) return PGX_OK;
  if (!col_idx || !src_eb || !tile_src || !mailbox || !has_bits ||
      (!dense && (!src_rs || !src_msg)) || (dense && !src_ids))
    return fail(PGX_EINVAL, "null scatter pointer");
  ScatterArgs a;
  a.col = col_idx;
  a.eb = src_eb;
  a.rs = src_rs;
  a.ids = src_ids;
  a.msg = src_msg;
  a.tile_src = tile_src;
  a.nsrc = nsrc;
  a.E = edges;
  a.mailbox = mailbox;
  a.has = has_bits;
  a.id_offset = id_offset;
  a.hub_ids = nullptr;
  a.nhubs = 0;
  a.cas_loop = 0;
  a.neutral = neutral;
  a.n = INT32_MAX;  // the slice ABI has no vertex count: unchecked
  a.peer_mb = reinterpret_cast<uint32_t *const *>(peer_mailboxes);
  a.bounds = bounds;
  a.world = world;
  a.lo = lo;
  a.hi = hi;
  const int64_t tiles = ceil_div(edges, kTile);
  int sms = 148, dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(tiles, kWarps),
                                                               (int64_t)sms * PGX_SCATTER_MIN_BLOCKS));
  cudaStream_t st = (cudaStream_t)stream;
  const size_t smem = scatter_smem(PGX_OP_MIN_U32);
  const int rf = g_opt[PGX_OPT_READ_FILTER];
  if (!dense) {
    PGX_CUDA(cudaFuncSetAttribute(scatter_kernel<PGX_OP_MIN_U32, MsgSrc::kFrontier, true>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    scatter_kernel<PGX_OP_MIN_U32, MsgSrc::kFrontier, true><<<grid, kBlock, smem, st>>>(a, rf);
  } else {
    PGX_CUDA(cudaFuncSetAttribute(scatter_kernel<PGX_OP_MIN_U32, MsgSrc::kSourceId, true>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    scatter_kernel<PGX_OP_MIN_U32, MsgSrc::kSourceId, true><<<grid, kBlock, smem, st>>>(a, rf);
  }
  PGX_CUDA(cudaGetLastError());
  return PGX_OK;
}

int pgx_scatter_peer_bfs(const int32_t *col_idx, const int32_t *src_eb, const int32_t *src_rs,
                         const void *src_msg, const int32_t *tile_src, int32_t nsrc,
                         int64_t edges, uint32_t *has_bits, const uint64_t *peer_has,
                         const int32_t *bounds, int32_t world, int32_t lo, int32_t hi,
                         uintptr_t stream) {
  if (edges < 0 || edges > INT32_MAX || nsrc < 0) return fail(PGX_EINVAL, "bad sizes");
  if (world < 1 || lo < 0 || hi < lo || !peer_has || !bounds)
    return fail(PGX_EINVAL, "bad peer arguments");
  if (edges == 0) return PGX_OK;
  if (!col_idx || !src_eb || !src_rs || !src_msg || !tile_src || !has_bits)
    return fail(PGX_EINVAL, "null scatter pointer");
  ScatterArgs a;
  memset(&a, 0, sizeof a);
  a.col = col_idx;
  a.eb = src_eb;
  a.rs = src_rs;
  a.msg = src_msg;
  a.tile_src = tile_src;
  a.nsrc = nsrc;
  a.E = edges;
  a.mailbox = nullptr;
  a.has = has_bits;
  a.neutral = kNeutralMin;
  a.n = INT32_MAX;
  a.peer_mb = reinterpret_cast<uint32_t *const *>(peer_has);
  a.bounds = bounds;
  a.world = world;
  a.lo = lo;
  a.hi = hi;
  const int64_t tiles = ceil_div(edges, kTile);
  int sms = 148, dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(tiles, kWarps),
                                                               (int64_t)sms * PGX_SCATTER_MIN_BLOCKS));
  cudaStream_t st = (cudaStream_t)stream;
  const size_t smem = scatter_smem(PGX_OP_MIN_U32);
  auto k = scatter_kernel<PGX_OP_MIN_U32, MsgSrc::kFrontier, true, true>;
  PGX_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k<<<grid, kBlock, smem, st>>>(a, 1);
  PGX_CUDA(cudaGetLastError());
  return PGX_OK;
}

int pgx_apply_slice_bfs(int32_t len, const int32_t *row_ptr, uint32_t *dist,
                        uint32_t *has_block, int32_t *f_eb, int32_t *f_rs, uint32_t *f_msg,
                        int32_t *tile_src, void *counters, int32_t count_only, uint32_t level,
                        uintptr_t stream) {
  if (len < 0 || !counters || (len && (!row_ptr || !dist || !has_block)))
    return fail(PGX_EINVAL, "bad apply_slice_bfs arguments");
  if (!len) return PGX_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const int grid = (int)ceil_div(len, kBlock * 4);
  apply_slice_bfs_kernel<<<grid, kBlock, 0, st>>>(len, row_ptr, dist, has_block, f_eb, f_rs,
                                                  f_msg, tile_src, (SliceCounters *)counters,
                                                  count_only, level);
  if (!count_only) {
    const int words = (int)ceil_div(len, 32);
    clear_words_kernel<<<(int)std::min<int64_t>(ceil_div(words, 256), 148 * 8), 256, 0, st>>>(
        has_block, words);
  }
  PGX_CUDA(cudaGetLastError());
  return PGX_OK;
}

int pgx_reset_touched(int32_t n, int32_t lo, int32_t hi, uint32_t *has_bits, uint32_t *mailbox,
                      uint32_t neutral, uintptr_t stream) {
  if (n < 1 || lo < 0 || hi < lo || hi > n || !has_bits || !mailbox)
    return fail(PGX_EINVAL, "bad pgx_reset_touched arguments");
  const int words = (int)ceil_div(n, 32);
  const int grid = (int)std::min<int64_t>(ceil_div(words, 256), 148 * 8);
  reset_touched_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(has_bits, n, lo, hi, mailbox,
                                                               neutral);
  PGX_CUDA(cudaGetLastError());
  return PGX_OK;
}

int pgx_peer_alloc(size_t bytes, void **ptr, void *ipc_handle) {
  if (!ptr || !bytes) return fail(PGX_EINVAL, "bad pgx_peer_alloc arguments");
  *ptr = nullptr;
  PGX_CUDA(cudaMalloc(ptr, bytes));
  if (ipc_handle) {
    cudaIpcMemHandle_t h;
    const cudaError_t e = cudaIpcGetMemHandle(&h, *ptr);
    if (e != cudaSuccess) {
      cudaFree(*ptr);
      *ptr = nullptr;
      return cuda_fail(e, "cudaIpcGetMemHandle");
    }
    memcpy(ipc_handle, &h, sizeof h);
  }
  return PGX_OK;
}

int pgx_peer_open(const void *ipc_handle, void **ptr) {
  if (!ipc_handle || !ptr) return fail(PGX_EINVAL, "bad pgx_peer_open arguments");
  cudaIpcMemHandle_t h;
  memcpy(&h, ipc_handle, sizeof h);
  *ptr = nullptr;
  PGX_CUDA(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return PGX_OK;
}

int pgx_peer_close(void *ptr) {
  if (!ptr) return fail(PGX_EINVAL, "null pointer");
  PGX_CUDA(cudaIpcCloseMemHandle(ptr));
  return PGX_OK;
}

int pgx_peer_free(void *ptr) {
  if (!ptr) return fail(PGX_EINVAL, "null pointer");
  PGX_CUDA(cudaFree(ptr));
  return PGX_OK;
}

int pgx_touched_scratch_bytes(int32_t n, size_t *bytes) {
  if (!bytes || n < 0) return fail(PGX_EINVAL, "bad arguments");
  *bytes = sizeof(int32_t) * (size_t)(ceil_div(ceil_div(n, 32), kCompactBlock) + 2);
  return PGX_OK;
}

int pgx_touched(int32_t n, int32_t lo, int32_t hi, const uint32_t *has_bits, uint32_t *mailbox,
                uint32_t neutral, uint64_t *pairs, int64_t *count, void *scratch,
                uintptr_t stream) {
  if (n < 1 || lo < 0 || hi < lo || hi > n || !has_bits || !count || !scratch ||
      (pairs && !mailbox))
    return fail(PGX_EINVAL, "bad pgx_touched arguments");
  const int words = (int)ceil_div(n, 32);
  const int nb = (int)ceil_div(words, kCompactBlock);
  cudaStream_t st = (cudaStream_t)stream;
  int32_t *blk = (int32_t *)scratch;
  touched_count_kernel<<<nb, kCompactBlock, 0, st>>>(has_bits, n, lo, hi, blk);
  touched_scan_kernel<<<1, kCompactBlock, 0, st>>>(blk, nb, count);
  if (pairs)
    touched_write_kernel<<<nb, kCompactBlock, 0, st>>>(has_bits, n, lo, hi, blk, mailbox, neutral,
                                                       (unsigned long long *)pairs);
  PGX_CUDA(cudaGetLastError());
  return PGX_OK;
}

int pgx_scatter_pairs(const uint64_t *pairs, int64_t count, uint32_t *mailbox, uintptr_t stream) {
  if (count < 0 || (count && (!pairs || !mailbox))) return fail(PGX_EINVAL, "bad pairs");
  if (!count) return PGX_OK;
  const int grid = (int)std::min<int64_t>(ceil_div(count, 256), 148 * 16);
  scatter_pairs_min_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(
      (const unsigned long long *)pairs, count, mailbox);
  PGX_CUDA(cudaGetLastError());
  return PGX_OK;
}

int pgx_slice_counters_bytes(size_t *bytes) {
  if (!bytes) return fail(PGX_EINVAL, "null out pointer");
  *bytes = sizeof(SliceCounters);
  return PGX_OK;
}

int pgx_apply_slice(int app, int32_t len, const int32_t *row_ptr, uint32_t *val,
                    uint32_t *mailbox_slice, int32_t *f_eb, int32_t *f_rs, uint32_t *f_msg,
                    int32_t *tile_src, void *counters, int32_t count_only, uint32_t neutral,
                    uint32_t *send_values, uintptr_t stream) {
  if (app != PGX_APP_CC && app != PGX_APP_SSSP) return fail(PGX_EINVAL, "min apps only");
  if (len < 0 || !counters) return fail(PGX_EINVAL, "bad apply_slice arguments");
  if (!len) return PGX_OK;
  const int grid = (int)ceil_div(len, kBlock * 4);
  cudaStream_t st = (cudaStream_t)stream;
  if (app == PGX_APP_CC)
    apply_slice_kernel<PGX_APP_CC><<<grid, kBlock, 0, st>>>(len, row_ptr, val, mailbox_slice, f_eb,
                                                           f_rs, f_msg, tile_src,
                                                           (SliceCounters *)counters, count_only,
                                                           neutral, send_values);
  else
    apply_slice_kernel<PGX_APP_SSSP><<<grid, kBlock, 0, st>>>(len, row_ptr, val, mailbox_slice,
                                                             f_eb, f_rs, f_msg, tile_src,
                                                             (SliceCounters *)counters,
                                                             count_only, neutral, nullptr);
  PGX_CUDA(cudaGetLastError());
  return PGX_OK;
}

int pgx_pr_apply_slice(int32_t len, const int32_t *row_ptr, double *rank, double *mailbox_slice,
                       double *share, double base, double damping, const double *dangling,
                       double n_total, int32_t last, double *partials, uintptr_t stream) {
  if (len < 0 || !(n_total >= 1.0) ||
      (len && (!row_ptr || !rank || !mailbox_slice || !share || !partials || !dangling)))
    return fail(PGX_EINVAL, "bad pr_apply_slice arguments");
  if (!len) return PGX_OK;
  const int grid = (int)ceil_div(len, kBlock);
  pr_apply_slice_kernel<<<grid, kBlock, 0, (cudaStream_t)stream>>>(
      len, row_ptr, rank, mailbox_slice, share, base, damping, dangling, n_total, last, partials);
  PGX_CUDA(cudaGetLastError());
  return PGX_OK;
}

int pgx_gather_slice(int32_t nrows, int64_t m, const int32_t *in_col, const void *in_graph_ws,
                     int32_t nsrc, const double *share, double *folded, double *head,
                     double *tail, uintptr_t stream) {
  if (nrows < 1 || m < 0 || m > INT32_MAX || nsrc < 0 || nsrc > nrows)
    return fail(PGX_EINVAL, "bad gather_slice sizes");
  if (!m) return PGX_OK;
  if (!in_col || !in_graph_ws || !share || !folded || !head || !tail)
    return fail(PGX_EINVAL, "null gather_slice pointer");
  if (reinterpret_cast<uintptr_t>(in_col) % 32)  // 256-bit id loads in the fold
    return fail(PGX_EINVAL, "in_col must be 32-byte aligned");
  GraphWs w;
  graph_ws_layout(nrows, m, &w, (char *)in_graph_ws);
  GatherArgs g;
  g.in_col = in_col;
  g.eb = w.nz_eb;
  g.ids = w.nz_id;
  g.tile_src = w.tile_src;
  g.nsrc = nsrc;  // the workspace header's non-zero row count (host copy)
  g.E = m;
  g.share = share;
  g.folded = folded;
  g.head = head;
  g.tail = tail;
  g.n = INT32_MAX;  // local source ids: unchecked
  cudaStream_t st = (cudaStream_t)stream;
  const size_t smem = (size_t)kWarps * kSlots * 8 + 16;
  int sms = 148, dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = (int)std::max<int64_t>(
      1, std::min<int64_t>(ceil_div(ceil_div(m, kTile), kWarps), (int64_t)sms * PGX_MIN_BLOCKS));
  PGX_CUDA(cudaFuncSetAttribute(gather_slice_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)smem));
  gather_slice_kernel<<<grid, kBlock, smem, st>>>(g);
  PGX_CUDA(cudaGetLastError());
  return PGX_OK;
}

int pgx_seg_scatter(int msg, const PgxSegIndex *seg, int64_t m, int32_t ndst, int32_t id_offset,
                    const uint32_t *send_values, uint32_t *mailbox, uint32_t *has_bits,
                    uint32_t neutral, unsigned *item_ctr, uintptr_t stream) {
  if (!seg || m < 1 || m > INT32_MAX || ndst < 1 || !mailbox || !has_bits || !item_ctr ||
      (msg == 1 && !send_values) || (msg != 0 && msg != 1))
    return fail(PGX_EINVAL, "bad pgx_seg_scatter arguments");
  if (seg->seg_log2 < 5 || seg->seg_log2 > kSegMaxLog2 || seg->nent < 1 || seg->nent > m ||
      seg->nitems < 1 || !seg->ent_src || !seg->col16 || !seg->tile_ent || !seg->items ||
      reinterpret_cast<uintptr_t>(seg->items) % 16 || reinterpret_cast<uintptr_t>(seg->col16) % 16)
    return fail(PGX_EINVAL, "malformed segmented index");
  SegPass sp;
  sp.ix = *seg;
  sp.m = m;
  sp.n = ndst;
  sp.snd = nullptr;
  sp.sv = send_values;
  sp.uniform = 0u;
  sp.mailbox = mailbox;
  sp.has = has_bits;
  sp.item_ctr = item_ctr;
  sp.write_mailbox = true;
  sp.id_offset = id_offset;
  sp.out_neutral = neutral;
  cudaStream_t st = (cudaStream_t)stream;
  PGX_CUDA(cudaMemsetAsync(item_ctr, 0, sizeof(unsigned), st));
  const size_t smem = seg_smem_bytes(seg->seg_log2) + 16;
  int sms = 148, dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = std::max(1, std::min(sms * PGX_MIN_BLOCKS, seg->nitems));
  if (msg == 0) {
    PGX_CUDA(cudaFuncSetAttribute(seg_slice_kernel<kSegSourceId>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    seg_slice_kernel<kSegSourceId><<<grid, kBlock, smem, st>>>(sp);
  } else {
    PGX_CUDA(cudaFuncSetAttribute(seg_slice_kernel<kSegLabel>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    seg_slice_kernel<kSegLabel><<<grid, kBlock, smem, st>>>(sp);
  }
  PGX_CUDA(cudaGetLastError());
  return PGX_OK;
}

int pgx_fold_spanning(int32_t nspan, const int32_t *rows, const int32_t *t0, const int32_t *t1,
                      const double *head, const double *tail, double *folded, uintptr_t stream) {
  if (nspan < 0 || (nspan && (!rows || !t0 || !t1 || !head || !tail || !folded)))
    return fail(PGX_EINVAL, "bad fold_spanning arguments");
  if (!nspan) return PGX_OK;
  const int grid = (int)std::min<int64_t>(ceil_div(nspan, 256), 148 * 8);
  fold_spanning_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(nspan, rows, t0, t1, head, tail,
                                                               folded);
  PGX_CUDA(cudaGetLastError());
  return PGX_OK;
}

int pgx_peer_enable(int32_t peer_device) {
  int dev = 0;
  PGX_CUDA(cudaGetDevice(&dev));
  if (peer_device == dev) return PGX_OK;
  const cudaError_t e = cudaDeviceEnablePeerAccess(peer_device, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();  // clear the sticky-free "already enabled" status
    return PGX_OK;
  }
  if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceEnablePeerAccess");
  return PGX_OK;
}

}  // extern "C"
