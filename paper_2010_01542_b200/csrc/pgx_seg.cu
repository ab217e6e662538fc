// pgx_seg.cu -- graph preparation for the segmented scatter (pgx_seg.cuh):
// the destination-segmented index of a CSR.
//
// An ENTRY is a maximal run of one source's edges whose destinations fall
// in one segment (2^seg_log2 consecutive vertex ids).  Rows are sorted
// (graph.py:185), so a row's runs are contiguous and appear in (source,
// segment) order along the CSR.  The index regroups the runs by segment,
// stably (sources stay ascending inside a segment):
//   1. runs: one warp per 256-edge tile maps its edges to their sources
//      (the pgx_graph_prepare tile map) and flags run starts -- a row start,
//      or a destination segment different from the previous edge's; per
//      tile counts, exclusive scan, then the runs are written in CSR order
//      (position, source, segment);
//   2. a stable LSD radix sort of the runs by segment (CUB, graph
//      preparation only);
//   3. entry edge offsets = exclusive scan of the sorted runs' lengths;
//      every run's destinations are copied as 16-bit segment offsets, the
//      first one flagged (bit 15: the scatter finds entry boundaries in
//      the destination stream itself);
//   4. the 256-edge tile map of the new edge order and the segments' edge
//      ranges, from which the host cuts the work items (hot segments into
//      slices, largest first).
// Every step is deterministic.
#include <cub/cub.cuh>

#include <vector>

#include "pgx_common.cuh"
#include "pgx_seg.cuh"

namespace pgx {
namespace {

constexpr int kRunWarps = 8;  // tiles per CTA of the run kernels

// EMIT = false: per-tile run counts; true: write the runs at tile_base.
template <bool EMIT>
__global__ void __launch_bounds__(kRunWarps * 32) seg_runs_kernel(
    int64_t m, const int32_t *__restrict__ col, GraphWs g, int L, int32_t *tile_cnt,
    const int32_t *tile_base, int32_t *run_pos, int32_t *run_src, uint32_t *run_key) {
  __shared__ int32_t s_eb[kRunWarps][kSlots];
  __shared__ int32_t s_id[kRunWarps][kSlots];
  const int lane = (int)lane_id(), warp = threadIdx.x >> 5;
  const int64_t ntiles = (m + kTile - 1) / kTile;
  const int64_t t = (int64_t)blockIdx.x * kRunWarps + warp;
  if (t >= ntiles) return;
  const int nsrc = g.hdr[0];
  const int i0 = g.tile_src[t];
  const int i1 = (t + 1 < ntiles) ? g.tile_src[t + 1] : nsrc - 1;
  const int k = i1 - i0 + 1;
  for (int j = lane; j < k; j += 32) {
    s_eb[warp][j] = g.nz_eb[i0 + j];
    s_id[warp][j] = g.nz_id[i0 + j];
  }
  __syncwarp();
  int base = EMIT ? tile_base[t] : 0;
  int cnt = 0;
  for (int r = 0; r < kItems; r++) {
    const int64_t e = t * kTile + r * 32 + lane;
    bool flag = false;
    int j = 0;
    uint32_t key = 0;
    if (e < m) {
      int lo = 0, hi = k - 1;  // last window source whose row starts <= e
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (s_eb[warp][mid] <= e) lo = mid;
        else hi = mid - 1;
      }
      j = lo;
      key = (uint32_t)col[e] >> L;
      flag = (e == s_eb[warp][j]) || (((uint32_t)col[e - 1] >> L) != key);
    }
    const unsigned b = __ballot_sync(0xFFFFFFFFu, flag);
    if (EMIT && flag) {
      const int q = base + __popc(b & lanemask_lt());
      run_pos[q] = (int32_t)e;
      run_src[q] = s_id[warp][j];
      run_key[q] = key;
    }
    base += __popc(b);
    cnt += __popc(b);
  }
  if (!EMIT && lane == 0) tile_cnt[t] = cnt;
}

__global__ void iota_kernel(int32_t *v, int64_t count) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x)
    v[i] = (int32_t)i;
}

// sorted entry i <- run r = perm[i]: source and length
__global__ void seg_entries_kernel(int64_t nent, const int32_t *perm, const int32_t *run_pos,
                                   const int32_t *run_src, int32_t *ent_src, int32_t *lens) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nent;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int r = perm[i];
    ent_src[i] = run_src[r];
    lens[i] = run_pos[r + 1] - run_pos[r];
  }
}

// the runs' destinations as 16-bit segment offsets, in segment order; the
// tile map of the new edge order
__global__ void seg_copy_kernel(int64_t nent, const int32_t *perm, const int32_t *run_pos,
                                const int32_t *__restrict__ col, const int32_t *ent_eb, int L,
                                uint16_t *col16, int32_t *tile_ent) {
  const uint32_t mask = (1u << L) - 1u;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nent;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int r = perm[i];
    const int32_t s = run_pos[r];
    const int32_t d0 = ent_eb[i], d1 = ent_eb[i + 1];
    // bit 15: the entry's first edge (the scatter's entry boundaries); the
    // offset is stored as its swizzled shared-memory slot (seg_swz)
    for (int32_t j = 0; j < d1 - d0; j++)
      col16[d0 + j] = (uint16_t)((uint32_t)seg_swz((int)((uint32_t)col[s + j] & mask)) |
                                 (j == 0 ? kSegEntryFlag : 0u));
    for (int64_t t = ((int64_t)d0 + kTile - 1) / kTile; t * kTile < d1; t++) tile_ent[t] = (int32_t)i;
  }
}

// seg_e[k] = first edge of segment k in the new order (seg_e[nseg] = m)
__global__ void seg_bounds_kernel(int64_t nent, const uint32_t *key, const int32_t *ent_eb,
                                  int32_t nseg, int64_t m, int32_t *seg_e) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nent;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t prev = i ? (int64_t)key[i - 1] : -1;
    for (int64_t k = prev + 1; k <= (int64_t)key[i]; k++) seg_e[k] = ent_eb[i];
    if (i == nent - 1)
      for (int64_t k = (int64_t)key[i] + 1; k <= nseg; k++) seg_e[k] = (int32_t)m;
  }
}

struct SegWs {
  int32_t *tile_cnt;  // [ntiles + 1], exclusive-scanned in place into tile_base
  int32_t *tile_base;
  int32_t *run_pos;   // [nent + 1]
  int32_t *run_src;   // [nent]
  uint32_t *key_in, *key_out;  // [nent]
  int32_t *val_in, *val_out;   // [nent]
  int32_t *lens;      // [nent + 1]
  int32_t *seg_e;     // [nseg + 1]
  void *temp;         // CUB temporary storage
  size_t temp_bytes;
};

int key_bits(int32_t nseg) {
  int b = 1;
  while ((1ll << b) < nseg) b++;
  return b;
}

size_t seg_ws_layout(int32_t ndst, int64_t m, int64_t nent, int L, SegWs *w, char *base) {
  size_t off = 0;
  auto take = [&](size_t bytes) {
    char *p = base ? base + off : nullptr;
    off += align_up(bytes);
    return p;
  };
  const int64_t ntiles = ceil_div(m, kTile);
  const int32_t nseg = (int32_t)ceil_div(ndst, (int64_t)1 << L);
  const int64_t ne = nent < 0 ? 0 : nent;
  SegWs x;
  x.tile_cnt = (int32_t *)take(sizeof(int32_t) * (ntiles + 1));
  x.tile_base = (int32_t *)take(sizeof(int32_t) * (ntiles + 1));
  x.run_pos = (int32_t *)take(sizeof(int32_t) * (ne + 1));
  x.run_src = (int32_t *)take(sizeof(int32_t) * (ne + 1));
  x.key_in = (uint32_t *)take(sizeof(uint32_t) * (ne + 1));
  x.key_out = (uint32_t *)take(sizeof(uint32_t) * (ne + 1));
  x.val_in = (int32_t *)take(sizeof(int32_t) * (ne + 1));
  x.val_out = (int32_t *)take(sizeof(int32_t) * (ne + 1));
  x.lens = (int32_t *)take(sizeof(int32_t) * (ne + 1));
  x.seg_e = (int32_t *)take(sizeof(int32_t) * (nseg + 1));
  size_t t1 = 0, t2 = 0, t3 = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, t1, (int32_t *)nullptr, (int32_t *)nullptr,
                                (int)(ntiles + 1));
  if (ne > 0) {
    cub::DeviceRadixSort::SortPairs(nullptr, t2, (uint32_t *)nullptr, (uint32_t *)nullptr,
                                    (int32_t *)nullptr, (int32_t *)nullptr, (int)ne, 0,
                                    key_bits(nseg));
    cub::DeviceScan::ExclusiveSum(nullptr, t3, (int32_t *)nullptr, (int32_t *)nullptr,
                                  (int)(ne + 1));
  }
  x.temp_bytes = std::max(t1, std::max(t2, t3)) + 256;
  x.temp = take(x.temp_bytes);
  if (w) *w = x;
  return off;
}

int seg_check(int32_t n, int64_t m, const int32_t *row_ptr, const int32_t *col_idx,
              const void *graph_ws, int32_t L) {
  int rc = check_graph(n, m, row_ptr, col_idx, graph_ws);
  if (rc) return rc;
  if (L < 5 || L > kSegMaxLog2) return fail(PGX_EINVAL, "seg_log2 must be in [5, 15]");
  if (m < 1) return fail(PGX_EINVAL, "the segmented index needs at least one edge");
  return PGX_OK;
}

int grid_for(int64_t count) {
  int64_t g = ceil_div(count, 256);
  return (int)std::max<int64_t>(1, std::min<int64_t>(g, 148 * 64));
}

// count the runs of every tile and scan them into tile_base; total -> *nent
int count_runs(int32_t n, int64_t m, const int32_t *col_idx, const void *graph_ws, int L,
               const SegWs &w, int64_t *nent, cudaStream_t st) {
  GraphWs g;
  graph_ws_layout(n, m, &g, (char *)graph_ws);
  const int64_t ntiles = ceil_div(m, kTile);
  seg_runs_kernel<false><<<(unsigned)ceil_div(ntiles, kRunWarps), kRunWarps * 32, 0, st>>>(
      m, col_idx, g, L, w.tile_cnt, nullptr, nullptr, nullptr, nullptr);
  PGX_CUDA(cudaGetLastError());
  PGX_CUDA(cudaMemsetAsync(w.tile_cnt + ntiles, 0, sizeof(int32_t), st));
  size_t tb = w.temp_bytes;
  PGX_CUDA(cub::DeviceScan::ExclusiveSum(w.temp, tb, w.tile_cnt, w.tile_base, (int)(ntiles + 1),
                                         st));
  int32_t total = 0;
  PGX_CUDA(cudaMemcpyAsync(&total, w.tile_base + ntiles, sizeof(int32_t), cudaMemcpyDeviceToHost,
                           st));
  PGX_CUDA(cudaStreamSynchronize(st));
  *nent = total;
  return PGX_OK;
}

}  // namespace
}  // namespace pgx

using namespace pgx;

extern "C" {

int pgx_seg_workspace_bytes(int32_t n, int64_t m, int64_t nent, int32_t seg_log2,
                            size_t *bytes) {
  if (!bytes || n < 1 || m < 0 || seg_log2 < 5 || seg_log2 > kSegMaxLog2 || nent > m)
    return fail(PGX_EINVAL, "bad segmented-index workspace arguments");
  *bytes = seg_ws_layout(n, m, nent, seg_log2, nullptr, nullptr);
  return PGX_OK;
}

int pgx_seg_max_items(int32_t n, int64_t m, int32_t seg_log2, int32_t *max_items) {
  if (!max_items || n < 1 || m < 0 || seg_log2 < 5 || seg_log2 > kSegMaxLog2)
    return fail(PGX_EINVAL, "bad segmented-index arguments");
  // one item per segment plus at most one extra slice per item target
  // (the target is >= m / kMaxSegSlices, see pgx_seg_build)
  *max_items = (int32_t)(ceil_div(n, (int64_t)1 << seg_log2) + kMaxSegSlices + 1);
  return PGX_OK;
}

int pgx_seg_count_ex(int32_t nrows, int32_t ndst, int64_t m, const int32_t *row_ptr,
                     const int32_t *col_idx, const void *graph_ws, int32_t seg_log2, void *ws,
                     size_t ws_bytes, int64_t *nent, uintptr_t stream) {
  int rc = seg_check(nrows, m, row_ptr, col_idx, graph_ws, seg_log2);
  if (rc) return rc;
  if (ndst < 1) return fail(PGX_EINVAL, "destination count must be >= 1");
  if (!ws || !nent) return fail(PGX_EINVAL, "null workspace / output");
  SegWs w;
  if (seg_ws_layout(ndst, m, -1, seg_log2, &w, (char *)ws) > ws_bytes)
    return fail(PGX_ENOMEM, "segmented-index workspace too small");
  return count_runs(nrows, m, col_idx, graph_ws, seg_log2, w, nent, (cudaStream_t)stream);
}

int pgx_seg_count(int32_t n, int64_t m, const int32_t *row_ptr, const int32_t *col_idx,
                  const void *graph_ws, int32_t seg_log2, void *ws, size_t ws_bytes,
                  int64_t *nent, uintptr_t stream) {
  return pgx_seg_count_ex(n, n, m, row_ptr, col_idx, graph_ws, seg_log2, ws, ws_bytes, nent,
                          stream);
}

int pgx_seg_build_ex(int32_t nrows, int32_t ndst, int64_t m, const int32_t *row_ptr,
                     const int32_t *col_idx, const void *graph_ws, int32_t seg_log2,
                     int64_t nent, void *ws, size_t ws_bytes, int32_t *ent_src, int32_t *ent_eb,
                     uint16_t *col16, int32_t *tile_ent, int32_t *items, int32_t *nitems,
                     int32_t ctas, uintptr_t stream) {
  int rc = seg_check(nrows, m, row_ptr, col_idx, graph_ws, seg_log2);
  if (rc) return rc;
  if (ndst < 1) return fail(PGX_EINVAL, "destination count must be >= 1");
  if (!ws || !ent_src || !ent_eb || !col16 || !tile_ent || !items || !nitems)
    return fail(PGX_EINVAL, "null segmented-index output");
  if (nent < 1 || nent > m) return fail(PGX_EINVAL, "entry count out of range");
  if (reinterpret_cast<uintptr_t>(items) % 16 || reinterpret_cast<uintptr_t>(col16) % 16 ||
      reinterpret_cast<uintptr_t>(ent_src) % 16)
    return fail(PGX_EINVAL, "items, col16 and ent_src must be 16-byte aligned");
  const int L = seg_log2;
  cudaStream_t st = (cudaStream_t)stream;
  SegWs w;
  if (seg_ws_layout(ndst, m, nent, L, &w, (char *)ws) > ws_bytes)
    return fail(PGX_ENOMEM, "segmented-index workspace too small");
  int64_t got = 0;
  rc = count_runs(nrows, m, col_idx, graph_ws, L, w, &got, st);
  if (rc) return rc;
  if (got != nent) return fail(PGX_EINVAL, "entry count does not match pgx_seg_count");
  GraphWs g;
  graph_ws_layout(nrows, m, &g, (char *)graph_ws);
  const int64_t ntiles = ceil_div(m, kTile);
  const int32_t nseg = (int32_t)ceil_div(ndst, (int64_t)1 << L);
  // 1. the runs in CSR order
  seg_runs_kernel<true><<<(unsigned)ceil_div(ntiles, kRunWarps), kRunWarps * 32, 0, st>>>(
      m, col_idx, g, L, nullptr, w.tile_base, w.run_pos, w.run_src, w.key_in);
  PGX_CUDA(cudaGetLastError());
  const int32_t m32 = (int32_t)m;
  PGX_CUDA(cudaMemcpyAsync(w.run_pos + nent, &m32, sizeof(int32_t), cudaMemcpyHostToDevice, st));
  iota_kernel<<<grid_for(nent), 256, 0, st>>>(w.val_in, nent);
  // 2. stable sort by segment
  size_t tb = w.temp_bytes;
  PGX_CUDA(cub::DeviceRadixSort::SortPairs(w.temp, tb, w.key_in, w.key_out, w.val_in, w.val_out,
                                           (int)nent, 0, key_bits(nseg), st));
  // 3. entries: sources, edge offsets, 16-bit destinations, tile map
  seg_entries_kernel<<<grid_for(nent), 256, 0, st>>>(nent, w.val_out, w.run_pos, w.run_src,
                                                     ent_src, w.lens);
  PGX_CUDA(cudaMemsetAsync(w.lens + nent, 0, sizeof(int32_t), st));
  tb = w.temp_bytes;
  PGX_CUDA(cub::DeviceScan::ExclusiveSum(w.temp, tb, w.lens, ent_eb, (int)(nent + 1), st));
  PGX_CUDA(cudaMemsetAsync(col16 + m, 0, sizeof(uint16_t) * kTile, st));
  seg_copy_kernel<<<grid_for(nent), 256, 0, st>>>(nent, w.val_out, w.run_pos, col_idx, ent_eb, L,
                                                  col16, tile_ent);
  const int32_t last = (int32_t)(nent - 1);
  PGX_CUDA(cudaMemcpyAsync(tile_ent + ntiles, &last, sizeof(int32_t), cudaMemcpyHostToDevice, st));
  // 4. segment edge ranges -> work items (host)
  seg_bounds_kernel<<<grid_for(nent), 256, 0, st>>>(nent, w.key_out, ent_eb, nseg, m, w.seg_e);
  PGX_CUDA(cudaGetLastError());
  std::vector<int32_t> se((size_t)nseg + 1);
  PGX_CUDA(cudaMemcpyAsync(se.data(), w.seg_e, sizeof(int32_t) * (nseg + 1),
                           cudaMemcpyDeviceToHost, st));
  PGX_CUDA(cudaStreamSynchronize(st));
  if (ctas <= 0) {
    int dev = 0, sms = 0;
    PGX_CUDA(cudaGetDevice(&dev));
    PGX_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    ctas = sms * PGX_MIN_BLOCKS;
  }
  // a hot segment is cut into slices of <= target edges so that the
  // largest items finish together (about kSegItemsPerCta items per CTA)
  const int64_t target = std::max<int64_t>(
      std::max<int64_t>(4096, ceil_div(m, kMaxSegSlices)), ceil_div(m, (int64_t)ctas * kSegItemsPerCta));
  struct Item { int32_t seg, e0, e1, sole; };
  std::vector<Item> v;
  for (int32_t k = 0; k < nseg; k++) {
    const int32_t a = se[k], b = se[k + 1];
    if (b <= a) continue;
    const int32_t sole = (b - a <= target) ? 1 : 0;
    for (int64_t x = a; x < b; x += target)
      v.push_back({k, (int32_t)x, (int32_t)std::min<int64_t>(b, x + target), sole});
  }
  std::stable_sort(v.begin(), v.end(), [](const Item &p, const Item &q) {
    return (p.e1 - p.e0) > (q.e1 - q.e0);
  });
  int32_t cap = 0;
  pgx_seg_max_items(ndst, m, L, &cap);
  if ((int64_t)v.size() > cap) return fail(PGX_EINVAL, "internal: too many work items");
  PGX_CUDA(cudaMemcpyAsync(items, v.data(), sizeof(Item) * v.size(), cudaMemcpyHostToDevice, st));
  PGX_CUDA(cudaStreamSynchronize(st));
  *nitems = (int32_t)v.size();
  return PGX_OK;
}

int pgx_seg_build(int32_t n, int64_t m, const int32_t *row_ptr, const int32_t *col_idx,
                  const void *graph_ws, int32_t seg_log2, int64_t nent, void *ws,
                  size_t ws_bytes, int32_t *ent_src, int32_t *ent_eb, uint16_t *col16,
                  int32_t *tile_ent, int32_t *items, int32_t *nitems, int32_t ctas,
                  uintptr_t stream) {
  return pgx_seg_build_ex(n, n, m, row_ptr, col_idx, graph_ws, seg_log2, nent, ws, ws_bytes,
                          ent_src, ent_eb, col16, tile_ent, items, nitems, ctas, stream);
}

}  // extern "C"
