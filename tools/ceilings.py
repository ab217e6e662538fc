"""Measure the scattered-access ceilings of the B200 (pgx_microbench) and
write them to profiles/ceilings_<tag>.json."""
import ctypes, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2010_01542_b200 import _lib

lib = _lib.load()
kinds = {"load_u32": 0, "load_f64": 1, "red_min_u32": 2, "red_add_f64": 3, "atom_min_u32": 4,
         "load_u32_cg": 5, "load_u32_l1_no_allocate": 6, "load_u32_relaxed_gpu": 7}
if len(sys.argv) > 2:
    kinds = {k: v for k, v in kinds.items() if k in sys.argv[2].split(",")}
out = {"gpu": torch.cuda.get_device_name(0), "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()),
       "how": "pgx_microbench: uniformly random slots (counter hash), 8 in flight/thread, "
              "148x8 CTAs x 256 threads, second launch timed with CUDA events", "results": []}
ops = 1 << 30
for size_mb in ((16,) if len(sys.argv) > 2 else (16, 64, 1024)):
    for name, k in kinds.items():
        elem = 8 if "f64" in name else 4
        n = (size_mb << 20) // elem
        buf = torch.zeros(n * elem, dtype=torch.uint8, device="cuda")
        if "min" in name:
            buf.fill_(255)
        ms = ctypes.c_float(0)
        _lib.check(lib.pgx_microbench(k, buf.data_ptr(), n, ops, 7, ctypes.byref(ms),
                                      torch.cuda.current_stream().cuda_stream), "pgx_microbench")
        rate = ops / (ms.value * 1e-3) / 1e9
        r = {"kind": name, "array_MiB": size_mb, "G_ops_per_s": round(rate, 1),
             "useful_GB_per_s": round(rate * elem, 1), "sector_GB_per_s": round(rate * 32, 1)}
        out["results"].append(r)
        print(r, flush=True)
        del buf
tag = sys.argv[1] if len(sys.argv) > 1 else "r1"
for d in ("profiles", "gpurun_out"):
    os.makedirs(d, exist_ok=True)
    with open(f"{d}/ceilings_{tag}.json", "w") as fh:
        json.dump(out, fh, indent=1)
