"""EXPERIMENT driver for tools/bin_exp.cu: propagation-blocked dense min
scatter (C2 superstep 0) vs the shipped pgx_scatter, bit-exact check."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2010_01542_b200 import _lib
from paper_2010_01542_b200.rmat import rmat_graph

SHIFT = 13
exp = ctypes.CDLL(os.environ.get("BINEXP", "exp/libbinexp.so"))
lib = _lib.load()
g = rmat_graph(sys.argv[1] if len(sys.argv) > 1 else "C2")
c = g.device_csr()
n, m = c.n, c.m
al = lambda x: (x + 255) // 256 * 256
o_id = al(16); o_eb = o_id + al(4 * (n + 1)); o_tile = o_eb + al(4 * (n + 1))
hdr = c.ws[:16].view(torch.int32)
nz_id = c.ws[o_id:o_id + 4 * (n + 1)].view(torch.int32)
nz_eb = c.ws[o_eb:o_eb + 4 * (n + 1)].view(torch.int32)
tile = c.ws[o_tile:o_tile + 4 * ((m + 255) // 256 + 2)].view(torch.int32)
nnz = int(hdr[0])
st = torch.cuda.current_stream().cuda_stream
P = ctypes.c_void_p
ev = lambda: torch.cuda.Event(enable_timing=True)

# reference: shipped dense scatter
mb_ref = torch.empty(n, dtype=torch.int32, device="cuda")
has_ref = torch.zeros(n // 32 + 2, dtype=torch.int32, device="cuda")
tr = []
for it in range(5):
    mb_ref.fill_(-1); has_ref.zero_()
    a, b = ev(), ev(); a.record()
    _lib.check(lib.pgx_scatter(0, 1, c.col_idx.data_ptr(), nz_eb.data_ptr(), None, nz_id.data_ptr(),
                               0, None, tile.data_ptr(), nnz, m, mb_ref.data_ptr(),
                               has_ref.data_ptr(), 0xFFFFFFFF, st), "pgx_scatter")
    b.record(); torch.cuda.synchronize(); tr.append(a.elapsed_time(b))

# binning
nbins = (n + (1 << SHIFT) - 1) >> SHIFT
indeg = torch.bincount(c.col_idx.to(torch.int64), minlength=n)
cap = torch.zeros(nbins, dtype=torch.int64, device="cuda")
cap.index_add_(0, torch.arange(n, device="cuda") >> SHIFT, indeg)
bin_base = torch.zeros(nbins + 1, dtype=torch.int64, device="cuda")
bin_base[1:] = torch.cumsum(cap, 0)
pairs = torch.empty(m * 2, dtype=torch.int32, device="cuda")
cursor = torch.zeros(nbins, dtype=torch.int32, device="cuda")
mb = torch.empty(n, dtype=torch.int32, device="cuda")
has = torch.zeros(n // 32 + 2, dtype=torch.int32, device="cuda")
chunk = int(os.environ.get("CHUNK", 16384))
ga, gb = int(os.environ.get("GRID_A", 296)), int(os.environ.get("GRID_B", 296))
ta, tb = [], []
for it in range(5):
    cursor.zero_(); mb.fill_(-1); has.zero_()
    a, b, d = ev(), ev(), ev(); a.record()
    rc = exp.binexp_phase_a(P(c.col_idx.data_ptr()), P(nz_eb.data_ptr()), P(nz_id.data_ptr()),
                            P(tile.data_ptr()), nnz, ctypes.c_int64(m), nbins,
                            P(bin_base.data_ptr()), P(cursor.data_ptr()), P(pairs.data_ptr()),
                            ga, ctypes.c_size_t(st))
    assert rc == 0, rc
    b.record(); torch.cuda.synchronize()
    cnt = cursor.to(torch.int64)
    assert bool((cnt <= cap).all())
    nch = (cnt + chunk - 1) // chunk
    bins = torch.repeat_interleave(torch.arange(nbins, device="cuda"), nch)
    first = torch.cumsum(nch, 0) - nch
    k = torch.arange(bins.numel(), device="cuda") - first[bins]
    lo = k * chunk
    hi = torch.minimum(lo + chunk, cnt[bins])
    items = torch.stack([bins, lo, hi, torch.zeros_like(bins)], 1).to(torch.int32).contiguous()
    a2 = ev(); a2.record()
    rc = exp.binexp_phase_b(P(pairs.data_ptr()), P(bin_base.data_ptr()), P(items.data_ptr()),
                            items.shape[0], n, P(mb.data_ptr()), P(has.data_ptr()), gb,
                            ctypes.c_size_t(st))
    assert rc == 0, rc
    d.record(); torch.cuda.synchronize()
    ta.append(a.elapsed_time(b)); tb.append(a2.elapsed_time(d))
med = lambda x: sorted(x[1:])[len(x[1:]) // 2]
print(f"m={m} nbins={nbins} items={items.shape[0]} chunk={chunk}")
print(f"pgx_scatter dense : {med(tr)*1e3:7.1f} us ({m/med(tr)/1e6:.1f} G/s)")
print(f"bin phase A       : {med(ta)*1e3:7.1f} us")
print(f"bin phase B       : {med(tb)*1e3:7.1f} us  (A+B {1e3*(med(ta)+med(tb)):.1f} us, "
      f"{m/(med(ta)+med(tb))/1e6:.1f} G/s)")
print("mailbox identical:", torch.equal(mb, mb_ref), " has identical:", torch.equal(has, has_ref))
