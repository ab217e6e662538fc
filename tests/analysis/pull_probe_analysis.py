"""CPU analysis behind the bottom-up SSSP probe order (K1p):
for C3's supersteps 1-4, how many in-row sources a vertex tests before its
first sender when it scans its (ascending) in-row from the front, from the
back, or alternating, and how many edges a probe budget of P leaves to the
remainder pass.  Uses the oracle's R-MAT generator and SSSP (test
infrastructure; runs here, no GPU).  usage: python tests/analysis/pull_probe_analysis.py"""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from oracle import oracle as O
t=time.time()
n, off, tgt = O.rmat_csr(O.RmatSpec(22, 16, .57, .19, .19, 3, False))
print("gen", time.time()-t, n, off[-1])
ioff, itgt = O.transpose(n, off, tgt)
src = int(np.argmax(np.diff(off)))
run = O.run_sssp(n, off, tgt, src)
dist = run.values
indeg = np.diff(ioff)
row = np.repeat(np.arange(n), indeg)
pos = np.arange(itgt.size) - ioff[row]
for s in range(1, 5):
    snd = (dist == s)
    hit = snd[itgt]
    E_s = int(np.diff(off)[snd].sum())
    # ascending: first hit index
    big = np.int64(1 << 40)
    first_asc = np.full(n, big); np.minimum.at(first_asc, row[hit], pos[hit])
    # descending
    rpos = indeg[row] - 1 - pos
    first_desc = np.full(n, big); np.minimum.at(first_desc, row[hit], rpos[hit])
    # two-ended: probe order lo0, hi0, lo1, hi1 ...: index of lo k = 2k, hi k = 2k+1
    tw = np.minimum(2 * pos, 2 * rpos + 1)
    first_two = np.full(n, big); np.minimum.at(first_two, row[hit], tw[hit])
    has = first_asc < big
    for name, f in (("asc", first_asc), ("desc", first_desc), ("two", first_two)):
        checks = np.where(f < big, f + 1, indeg).sum()
        # with probe prefix P then remainder whole
        res = [name, f"checks={checks/1e6:.1f}M"]
        for P in (1, 2, 4, 8):
            ok = f < P
            rem = np.where(~ok & (indeg > P), indeg - P, 0).sum()
            res.append(f"P{P}: hitfrac={ok.sum()/max(has.sum(),1):.3f} remE={rem/1e6:.2f}M")
        print(f"s{s} E_s={E_s/1e6:.1f}M F={snd.sum()} R={has.sum()}", *res)
