"""C5 (scale 26, 1.84e9 edges) on one GPU vs BASELINE.md section 3 known answers."""
import hashlib, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2010_01542_b200 as pgx
from paper_2010_01542_b200.rmat import rmat_graph

def sha(t, dt):
    h = hashlib.sha256()
    a = t.cpu().numpy().astype(dt, copy=False)
    h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()

t = time.time()
g = rmat_graph("C5")
torch.cuda.synchronize()
print(f"C5 generated on GPU: n={g.vertex_count} m={g.edge_count} in {time.time()-t:.1f}s, "
      f"mem {torch.cuda.max_memory_allocated()/2**30:.1f} GiB peak", flush=True)
ok = {}
ok["csr_off"] = sha(g.out_offsets, "<i8") == "f614c1f95e1a3306eb010a577c7da219b35785190bacf6375eb96f4532514738"
ok["csr_tgt"] = sha(g.out_targets, "<i4") == "7809334f406f147b22e18001f03fd95659dd863d8a4d96636ee0025d7d761880"
print("csr hashes", ok, flush=True)
prog = pgx.connected_components()
plan = pgx.plan_run(g, prog)
for i in range(3):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); plan.launch(); b.record(); torch.cuda.synchronize()
    rep = pgx.collect(plan, prog)
    E = sum(s.edges for s in rep.supersteps)
    print(f"run {i}: {a.elapsed_time(b):.2f} ms  GTEPS={E/a.elapsed_time(b)/1e6:.1f}", flush=True)
ok["labels"] = sha(torch.from_numpy(rep.values.astype(np.uint32)), "<u4") == \
    "2667f2ecc3e6e7cb00c5c53f2b8af394b2802cbd19de2a9e1b8122490b4b1154"
ok["active"] = [s.active_count for s in rep.supersteps] == [67108864, 31691446, 31654625, 24001955, 2770014, 15744, 43]
ok["bcast"] = [s.messages_sent for s in rep.supersteps] == [67108864, 28808188, 30736448, 3973129, 15743, 43, 0]
ok["edges"] = [s.edges for s in rep.supersteps] == [1844208942, 1838211760, 801105854, 5102558, 15802, 43, 0]
ok["components"] = len(np.unique(rep.values)) == 35429838
print("C5 known answers:", ok, "ALL OK" if all(ok.values()) else "MISMATCH")
for s in rep.supersteps:
    print(f"  s{s.index}: {s.seconds*1e6:9.1f} us act={s.active_count} F={s.messages_sent} E={s.edges}")
