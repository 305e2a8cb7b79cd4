"""Time and cross-check transfer-kernel variants (HDB_RESTRICT / HDB_PROLONG
modes; each mode in its own process since the library reads the knob once).

    python tools/transfer_variants.py            # driver: all modes
    python tools/transfer_variants.py --one      # child: current env
"""
import json
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def child():
    import hashlib
    import torch
    import paper_2412_04980_b200 as hdb  # noqa: F401
    from paper_2412_04980_b200 import _lib
    L = _lib.lib()
    out = {}
    for n in (4097, 1025, 513, 2049 + 1024):  # last: non-power-of-two fine size
        nc = (n - 1) // 2 + 1
        rng = np.random.default_rng(7)
        u = torch.from_numpy(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))).cuda()
        cu = torch.from_numpy(rng.standard_normal((nc, nc)) + 1j * rng.standard_normal((nc, nc))).cuda()
        c = torch.empty((nc, nc), dtype=torch.complex128, device="cuda")
        f = torch.empty((n, n), dtype=torch.complex128, device="cuda")
        fa = torch.empty((n, n), dtype=torch.complex128, device="cuda")
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

        def timeit(fn, reps=20):
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            ev0.record()
            for _ in range(reps):
                fn()
            ev1.record()
            torch.cuda.synchronize()
            return ev0.elapsed_time(ev1) / reps * 1e-3

        tr = timeit(lambda: _lib.check(L.hdb_restrict(u.data_ptr(), n, n, c.data_ptr(), 0)))
        _lib.check(L.hdb_restrict(u.data_ptr(), n, n, c.data_ptr(), 15))
        hz = hashlib.sha1(c.cpu().numpy().tobytes()).hexdigest()[:12]
        _lib.check(L.hdb_restrict(u.data_ptr(), n, n, c.data_ptr(), 0))
        hr = hashlib.sha1(c.cpu().numpy().tobytes()).hexdigest()[:12]
        tp = timeit(lambda: _lib.check(L.hdb_prolong(cu.data_ptr(), n, n, None, f.data_ptr())))
        hp = hashlib.sha1(f.cpu().numpy().tobytes()).hexdigest()[:12]
        ta = timeit(lambda: _lib.check(L.hdb_prolong(cu.data_ptr(), n, n, u.data_ptr(), fa.data_ptr())))
        ha = hashlib.sha1(fa.cpu().numpy().tobytes()).hexdigest()[:12]
        N = n * n
        out[n] = {"restrict_GBs": round(20 * N / tr / 1e9), "prolong_GBs": round(20 * N / tp / 1e9),
                  "prolong_acc_GBs": round(36 * N / ta / 1e9), "restrict_us": round(tr * 1e6, 1),
                  "prolong_us": round(tp * 1e6, 1), "acc_us": round(ta * 1e6, 1), "hash": [hr, hz, hp, ha]}
    print("RESULT " + json.dumps(out))


def main():
    modes = [("R3P3", {"HDB_RESTRICT": "3", "HDB_PROLONG": "3"}), ("R3P1", {"HDB_RESTRICT": "3", "HDB_PROLONG": "1"}),
             ("R0P0", {"HDB_RESTRICT": "0", "HDB_PROLONG": "0"})]
    for name, env in modes:
        e = dict(os.environ)
        e.update(env)
        r = subprocess.run([sys.executable, __file__, "--one"], env=e, capture_output=True, text=True)
        line = [x for x in r.stdout.splitlines() if x.startswith("RESULT ")]
        print(name, line[0][7:] if line else ("FAILED " + r.stderr[-2000:]), flush=True)


if __name__ == "__main__":
    child() if "--one" in sys.argv else main()
