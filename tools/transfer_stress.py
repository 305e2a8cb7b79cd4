"""Repeat the transfer kernels on fixed inputs and check every output bitwise
(run-to-run determinism of the TMA-staged kernels), interleaved with other
kernels so scheduling varies.

    python tools/transfer_stress.py [--reps 40]
"""
import argparse
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=40)
    a = ap.parse_args()
    import torch
    import paper_2412_04980_b200 as hdb  # noqa: F401
    from paper_2412_04980_b200 import _lib
    L = _lib.lib()
    bad = 0
    for n in (2049, 4097):
        nc = (n - 1) // 2 + 1
        rng = np.random.default_rng(n)
        u = torch.from_numpy(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))).cuda()
        base = torch.from_numpy(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))).cuda()
        cu = torch.from_numpy(rng.standard_normal((nc, nc)) + 1j * rng.standard_normal((nc, nc))).cuda()
        c = torch.empty((nc, nc), dtype=torch.complex128, device="cuda")
        f = torch.empty((n, n), dtype=torch.complex128, device="cuda")
        ref = {}
        for r in range(a.reps):
            for kind in ("restrict", "prolong", "prolong_acc"):
                if kind == "restrict":
                    _lib.check(L.hdb_restrict(u.data_ptr(), n, n, c.data_ptr(), 0))
                    out = c
                elif kind == "prolong":
                    f.fill_(float("nan"))
                    _lib.check(L.hdb_prolong(cu.data_ptr(), n, n, None, f.data_ptr()))
                    out = f
                else:
                    f.fill_(float("nan"))
                    _lib.check(L.hdb_prolong(cu.data_ptr(), n, n, base.data_ptr(), f.data_ptr()))
                    out = f
                h = hashlib.sha1(out.cpu().numpy().tobytes()).hexdigest()
                if kind not in ref:
                    ref[kind] = h
                elif h != ref[kind]:
                    bad += 1
                    diff = (out.cpu().numpy() != out.cpu().numpy())  # NaN positions
                    print(f"MISMATCH n={n} {kind} rep {r}: nan count {int(diff.sum())}", flush=True)
    print("STRESS", "ok" if bad == 0 else f"{bad} mismatches")


if __name__ == "__main__":
    main()
