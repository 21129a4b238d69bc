"""Driver for kout_micro.cu: times each variant on RMAT s24 (device-built)
with CUDA events, a 256 MiB L2 flush before every run, median of 7, and
checks that every union variant yields the same k-out partition.

  python profiles/micro/kout_micro.py [--scale 24]
"""
import argparse
import ctypes
import json
import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_2008_11839_b200 import build_csr, gen_rmat  # noqa: E402


def load():
    so = HERE / "kout_micro.so"
    if not so.exists():
        subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
                               "-Xcompiler", "-fPIC", "-shared", "-I", str(ROOT / "paper_2008_11839_b200/csrc"),
                               "-I", str(ROOT / "include"), str(HERE / "kout_micro.cu"), "-o", str(so)])
    return ctypes.CDLL(str(so))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=24)
    ap.add_argument("--reps", type=int, default=7)
    ap.add_argument("--cold", action="store_true", help="flush L2 after the set init too")
    a = ap.parse_args()
    lib = load()
    g = build_csr(gen_rmat(a.scale, 8, seed=1, device=True), keep_host=False)
    n, m = g.n, g.m
    off, tgt = g._d_off, g._d_tgt
    P = torch.empty(n, dtype=torch.int32, device="cuda")
    pairs = torch.empty(2 * n, dtype=torch.int32, device="cuda")
    sink = torch.zeros(1, dtype=torch.int32, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    vp = ctypes.c_void_p
    O, T, Pp, PR, S = vp(off.data_ptr()), vp(tgt.data_ptr()), vp(P.data_ptr()), vp(pairs.data_ptr()), vp(sink.data_ptr())
    lib.km_make_pairs(O, T, n, PR, st)

    def comps():
        x = P.long()
        while True:
            y = x[x]
            if torch.equal(y, x):
                return x
            x = y

    variants = {
        "stream": (False, lambda: lib.km_stream(O, T, n, S, st)),
        "rows": (True, lambda: lib.km_rows(Pp, O, T, n, st)),
        "make_pairs": (False, lambda: lib.km_make_pairs(O, T, n, PR, st)),
        "union_pairs": (True, lambda: lib.km_union_pairs(Pp, PR, n, st)),
        "rows_async_b4": (True, lambda: lib.km_rows_async(Pp, O, T, n, ctypes.c_int64(m), 4, 0, st)),
        "rows_async_b4_ef": (True, lambda: lib.km_rows_async(Pp, O, T, n, ctypes.c_int64(m), 4, 1, st)),
        "rows_async_b3_ef": (True, lambda: lib.km_rows_async(Pp, O, T, n, ctypes.c_int64(m), 3, 1, st)),
        "rows_bulk_b4": (True, lambda: lib.km_rows_bulk(Pp, O, T, n, ctypes.c_int64(m), 4, st)),
        "rows_bulk_b3": (True, lambda: lib.km_rows_bulk(Pp, O, T, n, ctypes.c_int64(m), 3, st)),
    }
    ref = None
    out = {"n": n, "m": m, "async_smem_per_block": lib.km_async_smem(), "bulk_smem_per_block": lib.km_bulk_smem()}
    for name, (uses_p, fn) in variants.items():
        ts = []
        for r in range(a.reps + 1):
            flush.fill_(r & 0xff)
            if uses_p:
                # as in the pipeline: the set init leaves P in L2 for the unions
                lib.km_init(Pp, n, st)
                if a.cold:
                    flush.fill_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            rc = fn()
            e1.record()
            torch.cuda.synchronize()
            assert rc == 0, (name, rc)
            if r:
                ts.append(e0.elapsed_time(e1))
        ts.sort()
        res = {"ms_median": ts[len(ts) // 2], "ms_min": ts[0]}
        if uses_p:
            c = comps()
            if ref is None:
                ref = c
            res["same_partition"] = bool(torch.equal(c, ref))
        out[name] = res
        print(name, res, flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
