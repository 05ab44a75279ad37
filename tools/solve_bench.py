#!/usr/bin/env python
"""Micro-benchmark of pba_solve_dense on synthetic SPD systems (banded and dense).

  python tools/solve_bench.py [--dim 5994] [--band 126] [--reps 5]
"""

import argparse
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2303_16878_b200 import native as N  # noqa: E402


def make_spd(dim, band, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    if band is None or band >= dim:
        A = torch.randn(dim, dim, dtype=torch.float64, device="cuda", generator=g)
        return A @ A.T + dim * torch.eye(dim, dtype=torch.float64, device="cuda")
    A = torch.randn(dim, dim, dtype=torch.float64, device="cuda", generator=g)
    A = torch.triu(torch.tril(A, band // 2), -(band // 2))
    return A @ A.T + 1e-3 * torch.eye(dim, dtype=torch.float64, device="cuda")


def run(dim, band, reps):
    lib = N.load()
    H = make_spd(dim, band)
    b = torch.randn(dim, dtype=torch.float64, device="cuda")
    work = torch.empty(int(lib.pba_solve_work_bytes(dim)), dtype=torch.uint8, device="cuda")
    delta = torch.zeros(dim, dtype=torch.float64, device="cuda")
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    stream = torch.cuda.current_stream().cuda_stream
    T = (dim + 63) // 64
    if band is None or band >= dim:
        env = np.zeros(T, np.int32)
    else:
        env = np.array([max(0, (t * 64 - band) // 64) for t in range(T)], np.int32)
    times = []
    for r in range(reps + 2):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        N.check(lib.pba_solve_dense(H.data_ptr(), b.data_ptr(), dim, 1e-3, env.ctypes.data,
                                    work.data_ptr(), delta.data_ptr(), st.data_ptr(), stream),
                "solve")
        e1.record()
        torch.cuda.synchronize()
        if r >= 2:
            times.append(e0.elapsed_time(e1))
    Hd = H.cpu().numpy()
    ref = np.linalg.solve(Hd + 1e-3 * np.diag(np.diag(Hd)), -b.cpu().numpy())
    err = np.abs(delta.cpu().numpy() - ref).max() / np.abs(ref).max()
    print(f"dim {dim} band {band}: {np.median(times):.3f} ms (status {int(st.item())}, rel err {err:.2e})")


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--dim", type=int, default=5994)
    ap.add_argument("--band", type=int, default=126)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--dense", action="store_true")
    a = ap.parse_args()
    run(a.dim, a.band, a.reps)
    if a.dense:
        run(2994, None, a.reps)
