"""Experiment driver for tools/seg_exp.cu: destination-segmented dense scatter
(CC superstep 0) vs the shipped pgx_scatter, same inputs, bit-exact check.

python tools/seg_probe.py C2 [seg_log2 ...]
"""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2010_01542_b200 import _lib
from paper_2010_01542_b200.rmat import rmat_graph

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
seg = ctypes.CDLL(os.path.join(ROOT, "exp", "libseg.so"))
seg.seg_scatter.restype = ctypes.c_int
P = ctypes.c_void_p
seg.seg_scatter.argtypes = [P, P, P, P, P, ctypes.c_int, ctypes.c_int, ctypes.c_int64, ctypes.c_int,
                            ctypes.c_int, P, P, P, ctypes.c_int, ctypes.c_int, ctypes.c_uint64]


def build(row_ptr, col, n, L, ctas):
    """Segment-grouped edge order: stable sort of the edges by destination
    segment (the CSR is source-major, so sources stay sorted inside one)."""
    m = col.numel()
    deg = (row_ptr[1:] - row_ptr[:-1])
    src = torch.repeat_interleave(torch.arange(n, dtype=torch.int32, device="cuda"), deg)
    sg = (col >> L).to(torch.int32)
    _, order = torch.sort(sg, stable=True)
    del _
    sgs = sg[order]
    del sg
    srcs = src[order]
    del src
    col16 = torch.cat([(col[order] & ((1 << L) - 1)).to(torch.int16), torch.zeros(256, dtype=torch.int16, device='cuda')])
    del order
    flag = torch.ones(m, dtype=torch.bool, device="cuda")
    flag[1:] = (srcs[1:] != srcs[:-1]) | (sgs[1:] != sgs[:-1])
    starts = torch.nonzero(flag).flatten()
    del flag
    ent_src = srcs[starts].contiguous()
    ent_eb = torch.cat([starts, torch.tensor([m], device="cuda")]).to(torch.int32)
    nseg = (n + (1 << L) - 1) >> L
    seg_e = torch.searchsorted(sgs, torch.arange(nseg + 1, dtype=torch.int32, device="cuda"))
    del sgs, srcs
    ntiles = (m + 255) // 256
    tstart = torch.arange(ntiles, dtype=torch.int64, device="cuda") * 256
    tile_ent = (torch.searchsorted(starts, tstart, right=True) - 1).to(torch.int32)
    tile_ent = torch.cat([tile_ent, tile_ent[-1:]])
    # work items: a segment, hot ones cut into slices of <= target edges
    target = max(4096, m // (ctas * int(os.environ.get('SEG_ITEMS', '2'))))
    se = seg_e.cpu().tolist()
    items = []
    for k in range(nseg):
        a, b = se[k], se[k + 1]
        sole = 1 if b - a <= target else 0
        while a < b:
            z = min(b, a + target)
            items.append((z - a, k, a, z, sole))
            a = z
    items.sort(key=lambda x: -x[0])  # largest first
    it = torch.tensor([x[1:] for x in items], dtype=torch.int32).flatten().cuda()
    return ent_src, ent_eb, col16.contiguous(), tile_ent, it, len(items), starts.numel()


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
    Ls = [int(x) for x in sys.argv[2:] if x.isdigit()] or [13, 14, 15]
    passes = [int(os.environ.get("SEG_PASS"))] if os.environ.get("SEG_PASS") else [4, 8]
    ctas_l = [int(os.environ.get("SEG_CTAS", "2"))]
    g = rmat_graph(cfg)
    c = g.device_csr()
    n, m = c.n, c.m
    lib = _lib.load()
    st = torch.cuda.current_stream().cuda_stream
    # ---- shipped scatter (reference result + time) ----
    al = lambda x: (x + 255) // 256 * 256
    o_id = al(16); o_eb = o_id + al(4 * (n + 1)); o_tile = o_eb + al(4 * (n + 1))
    hdr = c.ws[:16].view(torch.int32)
    nz_id = c.ws[o_id:o_id + 4 * (n + 1)].view(torch.int32)
    nz_eb = c.ws[o_eb:o_eb + 4 * (n + 1)].view(torch.int32)
    tile = c.ws[o_tile:o_tile + 4 * ((m + 255) // 256 + 2)].view(torch.int32)
    nnz = int(hdr[0])
    mb0 = torch.empty(n, dtype=torch.int32, device="cuda")
    has0 = torch.zeros(n // 32 + 2, dtype=torch.int32, device="cuda")
    ts = []
    for it in range(5):
        mb0.fill_(-1); has0.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        _lib.check(lib.pgx_scatter(0, 1, c.col_idx.data_ptr(), nz_eb.data_ptr(), None,
                                   nz_id.data_ptr(), 0, None, tile.data_ptr(), nnz, m,
                                   mb0.data_ptr(), has0.data_ptr(), 0xFFFFFFFF, st), "pgx_scatter")
        b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    t_ship = sorted(ts[1:])[len(ts[1:]) // 2]
    print(f"{cfg} n={n} m={m}: shipped dense scatter {t_ship*1e3:.1f} us "
          f"({m/t_ship/1e6:.1f} G edges/s)", flush=True)
    rp = c.row_ptr.to(torch.int64)
    for L in Ls:
        for ctas in ctas_l:
            t = time.time()
            ent_src, ent_eb, col16, tile_ent, items, nitems, nent = build(rp, c.col_idx, n, L, 148 * ctas)
            torch.cuda.synchronize()
            tb = time.time() - t
            mb = torch.empty(n, dtype=torch.int32, device="cuda")
            has = torch.zeros(n // 32 + 2, dtype=torch.int32, device="cuda")
            ctr = torch.zeros(1, dtype=torch.int32, device="cuda")
            for pas in passes:
                ts = []
                for it in range(5):
                    mb.fill_(-1); has.zero_(); ctr.zero_()
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record()
                    rc = seg.seg_scatter(ent_src.data_ptr(), ent_eb.data_ptr(), col16.data_ptr(),
                                         tile_ent.data_ptr(), items.data_ptr(), nitems, nent, m, n, L,
                                         mb.data_ptr(), has.data_ptr(), ctr.data_ptr(), ctas, pas, st)
                    b.record(); torch.cuda.synchronize()
                    assert rc == 0, rc
                    ts.append(a.elapsed_time(b))
                tt = sorted(ts[1:])[len(ts[1:]) // 2]
                ok_mb = torch.equal(mb, mb0)
                ok_has = torch.equal(has, has0)
                print(f"  S=2^{L} ctas/sm={ctas} pass={pas}: entries={nent} ({m/nent:.2f} edges/entry) "
                      f"items={nitems} build={tb:.2f}s  seg scatter {tt*1e3:.1f} us "
                      f"({m/tt/1e6:.1f} G edges/s, x{t_ship/tt:.2f})  mailbox_equal={ok_mb} has_equal={ok_has}",
                      flush=True)
            del ent_src, ent_eb, col16, tile_ent, items
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
