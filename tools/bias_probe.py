"""Developer probe: signed (bias) and rms relative error of the streaming products vs f64.

    python tools/bias_probe.py            # tensor-core path (default selection)
    OOCNMF_FORCE_FFMA=1 python tools/bias_probe.py

A one-signed mean relative error that grows with the reduction length points at the
accumulator rounding mode (truncation) rather than at the operand split.
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2202_09518_b200 import nmf  # noqa: E402


def main():
    tag = "ffma" if os.environ.get("OOCNMF_FORCE_FFMA") == "1" else "tc"
    for m, n, k in [(4096, 2048, 16), (4096, 4096, 32), (8192, 8192, 64), (2048, 16384, 32)]:
        rng = np.random.default_rng(m + n + k)
        a = rng.random((m, n), dtype=np.float32)
        w = rng.random((m, k)).astype(np.float32).astype(np.float64)
        h = rng.random((k, n)).astype(np.float32).astype(np.float64)
        with nmf.Context(0) as ctx:
            ctx.set_problem(m, n, k)
            ctx.load_dense(a)
            ctx.set_factors(w, h)
            aht, wta, _, _ = ctx.products()
        a64 = a.astype(np.float64)
        for name, got, ref in (("AHt", aht, a64 @ h.T), ("WtA", wta, w.T @ a64)):
            r = (got - ref) / ref
            print(f"{tag} m={m} n={n} k={k} {name}: mean {r.mean():+.3e} rms {np.sqrt((r * r).mean()):.3e}",
                  flush=True)


if __name__ == "__main__":
    main()
