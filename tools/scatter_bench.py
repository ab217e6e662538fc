"""Time the standalone pgx_scatter (dense CC superstep 0 of C2) in isolation."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2010_01542_b200 import _lib
from paper_2010_01542_b200.rmat import rmat_graph
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
mb = torch.empty(n, dtype=torch.int32, device="cuda")
has = torch.zeros(n // 32 + 2, dtype=torch.int32, device="cuda")
st = torch.cuda.current_stream().cuda_stream
ts = []
for it in range(6):
    mb.fill_(-1); has.zero_()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    _lib.check(lib.pgx_scatter(0, 1, c.col_idx.data_ptr(), nz_eb.data_ptr(), None, nz_id.data_ptr(),
                               0, None, tile.data_ptr(), nnz, m, mb.data_ptr(), has.data_ptr(),
                               0xFFFFFFFF, st),
               "pgx_scatter")
    b.record(); torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
t = sorted(ts[1:])[len(ts[1:]) // 2]
print(f"{os.environ.get('PGX_LIB','default')}: dense scatter m={m}: {t*1e3:.1f} us = {m/t/1e6:.1f} G edges/s")
