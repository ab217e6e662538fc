// pgx_graph.cu -- graph preparation (int32 row pointers, the compacted
// sender list, the 256-edge tile map), the R-MAT input generator, and the
// library-wide C ABI (version, errors, options).
#include "pgx_common.cuh"

namespace pgx {

thread_local std::string g_last_error;

// tuning knobs (pgx_set_option); defaults are the shipped configuration
int g_opt[PGX_OPT_COUNT] = {
    /* PGX_OPT_READ_FILTER */ 1,
    /* PGX_OPT_CTAS_PER_SM */ 0,   // 0 = occupancy maximum
    /* PGX_OPT_CAS_LOOP */ 0,      // ablation: CAS retry per message
    /* PGX_OPT_VERTEX_SCHED */ 0,  // ablation: one thread per sender
    /* PGX_OPT_LAYOUT */ PGX_LAYOUT_EXTERNALISED,
    /* PGX_OPT_SEG_MIN_EDGES */ 256,  // segmented scatter from m/4 sender edges
    /* PGX_OPT_SEG_PREDICT */ 1,      // skip the frontier before predicted segmented supersteps
    /* PGX_OPT_PULL_MIN_EDGES */ 128, // unit-weight SSSP bottom-up from m/8 sender edges
};

namespace {

// ------------------------------------------------------------------
// graph preparation kernels: order-preserving compaction of the vertices
// with out-degree > 0 (warp ballot + block scan), then the tile map
// ------------------------------------------------------------------

__global__ void offsets_to_i32_kernel(const int64_t *in, int32_t *out, int64_t count) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (int32_t)in[i];
}

__global__ void nz_count_kernel(const int32_t *row_ptr, int32_t n, int32_t *blk) {
  __shared__ int s_warp[33];
  const int64_t v = blockIdx.x * (int64_t)kCompactBlock + threadIdx.x;
  const int f = (v < n && row_ptr[v + 1] > row_ptr[v]) ? 1 : 0;
  int total;
  block_excl_scan(f, s_warp, &total);
  if (threadIdx.x == 0) blk[blockIdx.x] = total;
}

__global__ void nz_scan_blocks_kernel(int32_t *blk, int32_t nb, int32_t *hdr) {
  // single CTA: exclusive scan of per-block counts
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
  if (threadIdx.x == 0) {
    blk[nb] = carry;
    hdr[0] = carry;
  }
}

__global__ void nz_write_kernel(const int32_t *row_ptr, int32_t n, const int32_t *blk,
                                int32_t *nz_id, int32_t *nz_eb, int64_t m) {
  __shared__ int s_warp[33];
  const int64_t v = blockIdx.x * (int64_t)kCompactBlock + threadIdx.x;
  const int f = (v < n && row_ptr[v + 1] > row_ptr[v]) ? 1 : 0;
  int total;
  const int ex = block_excl_scan(f, s_warp, &total);
  if (f) {
    const int pos = blk[blockIdx.x] + ex;
    nz_id[pos] = (int32_t)v;
    nz_eb[pos] = row_ptr[v];
  }
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) nz_eb[blk[gridDim.x]] = (int32_t)m;
}

__global__ void tile_map_kernel(const int32_t *hdr, const int32_t *nz_eb, int32_t *tile_src) {
  const int nnz = hdr[0];
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nnz; i += gridDim.x * blockDim.x) {
    const int64_t eb = nz_eb[i], ee = nz_eb[i + 1];
    for (int64_t t = (eb + kTile - 1) / kTile; t * kTile < ee; t++) tile_src[t] = i;
  }
}

// ------------------------------------------------------------------
// R-MAT generator, input construction only
// ------------------------------------------------------------------

__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void rmat_kernel(int scale, int64_t first, int64_t count, uint64_t ta, uint64_t tab,
                            uint64_t tabc, uint64_t base, int symmetric, int64_t lo, int64_t hi,
                            unsigned long long *keys, int64_t capacity,
                            unsigned long long *counter) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < count;
       k += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t i = (uint64_t)(first + k);
    uint64_t s = 0, d = 0;
    for (int l = 0; l < scale; l++) {
      const uint64_t r = splitmix64(base + i * (uint64_t)scale + (uint64_t)l) >> 11;
      const int q = r < ta ? 0 : r < tab ? 1 : r < tabc ? 2 : 3;
      const int bit = scale - 1 - l;
      s |= (uint64_t)(q >> 1) << bit;
      d |= (uint64_t)(q & 1) << bit;
    }
    if (s == d) continue;
    const bool fwd = (int64_t)s >= lo && (int64_t)s < hi;
    const bool rev = symmetric && (int64_t)d >= lo && (int64_t)d < hi;
    const int cnt = (fwd ? 1 : 0) + (rev ? 1 : 0);
    if (!cnt) continue;
    unsigned long long pos = atomicAdd(counter, (unsigned long long)cnt);
    if (fwd && (int64_t)pos < capacity) keys[pos++] = (s << 32) | d;
    if (rev && (int64_t)pos < capacity) keys[pos] = (d << 32) | s;
  }
}


}  // namespace
}  // namespace pgx

using namespace pgx;

extern "C" {

int pgx_abi_version(void) { return PGX_ABI_VERSION; }

const char *pgx_last_error(void) { return g_last_error.c_str(); }


int pgx_set_option(int key, int value) {
  if (key < 0 || key >= PGX_OPT_COUNT) return fail(PGX_EINVAL, "unknown option");
  g_opt[key] = value;
  return PGX_OK;
}

int pgx_device_sm_count(int device, int *sm_count) {
  if (!sm_count) return fail(PGX_EINVAL, "null out pointer");
  PGX_CUDA(cudaDeviceGetAttribute(sm_count, cudaDevAttrMultiProcessorCount, device));
  return PGX_OK;
}

int pgx_offsets_to_i32(const int64_t *offsets64, int32_t *row_ptr, int64_t count,
                       uintptr_t stream) {
  if (count < 0 || (count && (!offsets64 || !row_ptr))) return fail(PGX_EINVAL, "bad offsets");
  if (!count) return PGX_OK;
  const int grid = (int)std::min<int64_t>(ceil_div(count, 256), 148 * 16);
  offsets_to_i32_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(offsets64, row_ptr, count);
  PGX_CUDA(cudaGetLastError());
  return PGX_OK;
}

int pgx_graph_workspace_bytes(int64_t n, int64_t m, size_t *bytes) {
  if (!bytes || n < 0 || m < 0) return fail(PGX_EINVAL, "bad sizes");
  *bytes = graph_ws_layout(n, m, nullptr, nullptr);
  return PGX_OK;
}

int pgx_graph_prepare(int32_t n, int64_t m, const int32_t *row_ptr, void *graph_ws,
                      size_t graph_ws_bytes, uintptr_t stream) {
  if (n < 1 || m < 0 || m > INT32_MAX || !row_ptr || !graph_ws)
    return fail(PGX_EINVAL, "bad graph_prepare arguments");
  GraphWs g;
  if (graph_ws_layout(n, m, &g, (char *)graph_ws) > graph_ws_bytes)
    return fail(PGX_ENOMEM, "graph workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  const int nb = (int)ceil_div(n, kCompactBlock);
  nz_count_kernel<<<nb, kCompactBlock, 0, st>>>(row_ptr, n, g.blk);
  nz_scan_blocks_kernel<<<1, kCompactBlock, 0, st>>>(g.blk, nb, g.hdr);
  nz_write_kernel<<<nb, kCompactBlock, 0, st>>>(row_ptr, n, g.blk, g.nz_id, g.nz_eb, m);
  int sms = 148;
  int dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  tile_map_kernel<<<sms * 8, 256, 0, st>>>(g.hdr, g.nz_eb, g.tile_src);
  PGX_CUDA(cudaGetLastError());
  return PGX_OK;
}

int pgx_rmat_keys(int32_t scale, int64_t first_draw, int64_t num_draws, double a, double b,
                  double c, uint64_t seed, int32_t symmetric, int64_t src_lo, int64_t src_hi,
                  uint64_t *keys, int64_t capacity, int64_t *count, uintptr_t stream) {
  if (scale < 1 || scale > 30 || num_draws < 0 || !keys || !count)
    return fail(PGX_EINVAL, "bad R-MAT arguments");
  if (!num_draws) return PGX_OK;
  const double two53 = 9007199254740992.0;
  const uint64_t ta = (uint64_t)floor(a * two53);
  const uint64_t tab = (uint64_t)floor((a + b) * two53);
  const uint64_t tabc = (uint64_t)floor((a + b + c) * two53);
  uint64_t z = seed + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  const uint64_t base = z ^ (z >> 31);
  const int grid = (int)std::min<int64_t>(ceil_div(num_draws, 256), 148 * 32);
  rmat_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(
      scale, first_draw, num_draws, ta, tab, tabc, base, symmetric, src_lo, src_hi,
      (unsigned long long *)keys, capacity, (unsigned long long *)count);
  PGX_CUDA(cudaGetLastError());
  return PGX_OK;
}

}  // extern "C"
