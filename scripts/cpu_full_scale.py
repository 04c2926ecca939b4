"""The unmodified reference (oracle/_ref) at the FULL sizes of BASELINE
configs 1-3 (BASELINE.md §2's host plan), one step each, on this host's
cores — the bench's cpu_baseline times bounded samples instead, so that the
default run stays within minutes. Records the CPU model, core count and RAM.

  python scripts/cpu_full_scale.py > profiles/r02_cpu_full_scale.json
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import oracle  # noqa: E402


def main():
    lib, port = oracle.Ref(), oracle.Port()
    threads = os.cpu_count() or 1
    host = bench.host_info() if hasattr(bench, "host_info") else {}
    for config in (1, 2, 3):
        t0 = time.perf_counter()
        if config == 1:
            full = port.gen_uniform(1, 1 << 20, 1 << 20, 16)
        elif config == 2:
            full = port.gen_rmat(7, 22, 16 << 22)
        else:
            full = port.gen_hypersparse(5, 1 << 22, 1 << 22, 2 << 22)
        m, n = full.shape
        r, c, v = full.arrays()
        coo = lib.from_coo(m, n, r, c, v)
        if config == 3:
            b = port.gen_dense(3, n * 64).reshape(n, 64)
        else:
            x = port.gen_dense(3, n)
        gen_s = time.perf_counter() - t0
        t0 = time.perf_counter()
        if config == 1:
            a = lib.convert(coo, "CSR")
            t1 = time.perf_counter()
            lib.spmv(a, x, threads=threads)
        elif config == 2:
            sel, rem, _ = lib.decompose_rows(coo, bench.Cfg2.threshold)
            e, co = lib.convert(rem, "ELL"), lib.convert(sel, "COO")
            t1 = time.perf_counter()
            lib.spmv(e, x, threads=threads) + lib.spmv(co, x, threads=threads)
        else:
            a = lib.convert(coo, "DCSR")
            lib.convert(coo, "CSC")
            t1 = time.perf_counter()
            lib.spmm(a, b, threads=threads)
        t2 = time.perf_counter()
        print(json.dumps({"config": config, "impl": "reference (oracle/_ref, unmodified headers)", "rows": m, "cols": n,
                          "nnz": len(v), "step_s": round(t2 - t0, 3), "convert_s": round(t1 - t0, 3),
                          "kernel_s": round(t2 - t1, 3), "Mnnz_per_s": round(len(v) / (t2 - t0) / 1e6, 4),
                          "threads_run_kernel": threads, "conversions": "single-threaded (as in the reference)",
                          "generate_s": round(gen_s, 1), "host": host}), flush=True)


if __name__ == "__main__":
    main()
