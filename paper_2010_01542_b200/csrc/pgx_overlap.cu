// pgx_overlap.cu -- connected components from host memory: superstep 0
// scattered chunk by chunk while the CSR is being uploaded.
//
// In superstep 0 every vertex sends its own id along its out-edges
// (algorithms.py:99-108; engine.py:255-316 runs it as the first superstep),
// so the messages of an edge range depend on nothing but the range: the
// host uploads the offsets (and builds the tile map), then copies the
// targets in chunks on a copy stream while this kernel combines each
// landed chunk into the run's mailbox / has-bitmask.  The persistent CC
// kernel then starts with the apply of superstep 0
// (pgx_cc_run_prescattered, min_run_kernel<..., PRE = true>).  The mailbox
// and has-bitmask end up exactly as K1's superstep 0 leaves them: a
// read-filtered red.min per message, the has bit set by every lane whose
// filter read saw the neutral (the first publication of a slot).
#include "pgx_common.cuh"

namespace pgx {
namespace {

constexpr int kOvBlock = 256;
constexpr int kOvWarps = kOvBlock / 32;

// one warp per 256-edge tile of [e_lo, e_hi): the tile's row starts / ids
// staged in shared memory, 8 edges per lane (coalesced target loads), the
// source of each edge found by binary search over the staged row starts
__global__ void __launch_bounds__(kOvBlock) cc_source_scatter_kernel(
    const int32_t *col, GraphWs g, int64_t m, int64_t e_lo, int64_t e_hi, uint32_t *mailbox,
    uint32_t *has, int32_t n) {
  __shared__ int32_t s_eb[kOvWarps][kSlots];
  __shared__ int32_t s_id[kOvWarps][kSlots];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t ntiles = (m + kTile - 1) / kTile;
  const int32_t nsrc = g.hdr[0];
  const int64_t t_lo = e_lo / kTile, t_hi = (e_hi + kTile - 1) / kTile;
  for (int64_t t = t_lo + (int64_t)blockIdx.x * kOvWarps + warp; t < t_hi;
       t += (int64_t)gridDim.x * kOvWarps) {
    const int64_t e0 = t * kTile;
    const int64_t a = max(e0, e_lo), b = min(min(e0 + kTile, m), e_hi);
    const int i0 = g.tile_src[t];
    const int i1 = (t + 1 < ntiles) ? g.tile_src[t + 1] : nsrc - 1;
    const int k = i1 - i0 + 1;
    __syncwarp();
    for (int j = lane; j <= k; j += 32) {
      const int i = i0 + j;
      if (j < k) {
        s_eb[warp][j] = g.nz_eb[i];
        s_id[warp][j] = g.nz_id[i];
      } else {
        s_eb[warp][j] = (i < nsrc) ? g.nz_eb[i] : (int32_t)m;
      }
    }
    __syncwarp();
#pragma unroll 4
    for (int r = 0; r < kTile / 32; r++) {
      const int64_t e = e0 + r * 32 + lane;
      if (e < a || e >= b) continue;
      int lo = 0, hi = k;  // largest row with start <= e
      while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if ((int64_t)s_eb[warp][mid] <= e) lo = mid; else hi = mid;
      }
      const uint32_t src = (uint32_t)s_id[warp][lo];
      const int32_t dst = col[e];
      PGX_ASSERT(dst >= 0 && dst < n);
      const uint32_t old = mailbox[dst];
      if (src < old) {
        red_min_u32(mailbox + dst, src);
        if (old == kNeutralMin) red_or_b32(has + (dst >> 5), 1u << (dst & 31));
      }
    }
  }
}

}  // namespace
}  // namespace pgx

using namespace pgx;

extern "C" {

int pgx_cc_prescatter_init(int32_t n, int64_t m, int32_t max_supersteps, void *run_ws,
                           size_t run_ws_bytes, uintptr_t stream) {
  if (n < 1 || m < 0 || max_supersteps < 1 || !run_ws)
    return fail(PGX_EINVAL, "bad pre-scatter arguments");
  RunWs w;
  if (run_ws_layout(PGX_APP_CC, n, m, max_supersteps, &w, (char *)run_ws) > run_ws_bytes)
    return fail(PGX_ENOMEM, "run workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  PGX_CUDA(cudaMemsetAsync(w.mailbox, 0xFF, sizeof(uint32_t) * (size_t)n, st));  // neutral
  PGX_CUDA(cudaMemsetAsync(w.has, 0, sizeof(uint32_t) * (size_t)(n / 32 + 2), st));
  return PGX_OK;
}

int pgx_cc_source_scatter(int32_t n, int64_t m, const int32_t *row_ptr, const int32_t *col_idx,
                          const void *graph_ws, int64_t e_lo, int64_t e_hi,
                          int32_t max_supersteps, void *run_ws, size_t run_ws_bytes,
                          uintptr_t stream) {
  int rc = check_graph(n, m, row_ptr, col_idx, graph_ws);
  if (rc) return rc;
  if (e_lo < 0 || e_hi < e_lo || e_hi > m) return fail(PGX_EINVAL, "edge range out of bounds");
  if (max_supersteps < 1 || !run_ws) return fail(PGX_EINVAL, "bad pre-scatter arguments");
  RunWs w;
  if (run_ws_layout(PGX_APP_CC, n, m, max_supersteps, &w, (char *)run_ws) > run_ws_bytes)
    return fail(PGX_ENOMEM, "run workspace too small");
  if (e_hi == e_lo) return PGX_OK;
  GraphWs g;
  graph_ws_layout(n, m, &g, (char *)graph_ws);
  const int64_t tiles = (e_hi + kTile - 1) / kTile - e_lo / kTile;
  int sms = 148, dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = (int)std::max<int64_t>(
      1, std::min<int64_t>((tiles + kOvWarps - 1) / kOvWarps, (int64_t)sms * 8));
  cc_source_scatter_kernel<<<grid, kOvBlock, 0, (cudaStream_t)stream>>>(
      col_idx, g, m, e_lo, e_hi, reinterpret_cast<uint32_t *>(w.mailbox), w.has, n);
  PGX_CUDA(cudaGetLastError());
  return PGX_OK;
}

}  // extern "C"
