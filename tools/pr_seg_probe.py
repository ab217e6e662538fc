"""Experiment driver for tools/pr_seg_exp.cu (PageRank fold as a
destination-segmented push with shared-memory f64 sums) vs the shipped
pull fold (pgx_gather_slice over the in-CSR), one fold on C4.
usage: pr_seg_probe.py C4 [seg_log2 ...]"""
import ctypes, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2010_01542_b200 as pgx
from paper_2010_01542_b200 import _lib
from paper_2010_01542_b200.rmat import rmat_graph

so = os.path.join(ROOT, "exp", "libprseg.so")
os.makedirs(os.path.dirname(so), exist_ok=True)
subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared",
                "-Xcompiler", "-fPIC", "-I", os.path.join(ROOT, "include"), "-o", so,
                os.path.join(ROOT, "tools", "pr_seg_exp.cu")], check=True)
E = ctypes.CDLL(so)
E.pr_seg_fold.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p,
                          ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                          ctypes.c_size_t]
cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
Ls = [int(x) for x in sys.argv[2:]] or [12, 13]
g = rmat_graph(cfg)
csr = g.device_csr()
n, m = csr.n, csr.m
st = torch.cuda.current_stream()
deg = torch.diff(csr.row_ptr).to(torch.float64)
share = torch.where(deg > 0, (1.0 / n) / deg.clamp(min=1), torch.zeros_like(deg))
src = torch.repeat_interleave(torch.arange(n, device="cuda"), torch.diff(csr.row_ptr).long())
ref = torch.zeros(n, dtype=torch.float64, device="cuda").index_add_(0, csr.col_idx.long(), share[src])
del src


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in ev:
        a.record(); fn(); b.record()
    torch.cuda.synchronize()
    return sorted(a.elapsed_time(b) for a, b in ev)[reps // 2]


# the shipped pull fold (gather kernel alone; tile-spanning rows not combined)
csr.ensure_transpose(st)
lib = _lib.load()
nsrc = int(csr.in_ws[:16].view(torch.int32)[0])
folded = torch.zeros(n, dtype=torch.float64, device="cuda")
ntile = (m + 255) // 256 + 2
head = torch.zeros(ntile, dtype=torch.float64, device="cuda")
tail = torch.zeros(ntile, dtype=torch.float64, device="cuda")
pull_ms = timed(lambda: _lib.check(lib.pgx_gather_slice(n, m, csr.in_col.data_ptr(), csr.in_ws.data_ptr(), nsrc,
                                                        share.data_ptr(), folded.data_ptr(), head.data_ptr(),
                                                        tail.data_ptr(), st.cuda_stream), "gather"))
print(f"{cfg} pull fold (gather kernel): {pull_ms:.3f} ms  {m / pull_ms / 1e6:.1f} G in-edges/s", flush=True)
for L in Ls:
    csr.seg, csr.seg_arrays = None, ()
    csr.ensure_segments(st, seg_log2=L)
    ix = csr.seg
    ctr = torch.zeros(1, dtype=torch.int32, device="cuda")
    out = torch.zeros(n, dtype=torch.float64, device="cuda")

    def run():
        ctr.zero_()
        out.zero_()
        rc = E.pr_seg_fold(ctypes.byref(ix), m, n, share.data_ptr(), out.data_ptr(), ctr.data_ptr(), 0, 296,
                           st.cuda_stream)
        assert rc == 0
    ms = timed(run)
    err = float(((out - ref).abs() / ref.abs().clamp(min=1e-300)).max())
    print(f"{cfg} push-seg L={L}: {ms:.3f} ms  {m / ms / 1e6:.1f} G edges/s  entries={ix.nent} "
          f"({m / ix.nent:.2f} edges/entry)  max rel err vs index_add {err:.2e}", flush=True)
