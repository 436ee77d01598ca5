"""Small cases of every engine for compute-sanitizer (memcheck / racecheck / synccheck / initcheck).

    compute-sanitizer --tool memcheck python tools/sanitize_cases.py [engine ...]

Each case runs leg2cheb and cheb2leg through the C ABI (lc_execute, twice on one plan so that the
re-armed flags and counters are exercised, and once through lc_execute_host) and checks the result
against the CPU oracle, so a sanitizer run that passes also computed the right answer.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
from lc_inputs import batch  # noqa: E402
from paper_2411_00033_b200 import Plan  # noqa: E402

CASES = {1: [(3000, 3), (70001, 1)], 2: [(3000, 16), (1500, 9)], 3: [(40000, 8), (9000, 11)]}


def main(engines):
    dev = torch.device("cuda", 0)
    for eng in engines:
        for n, V in CASES[eng]:
            x = batch("normal", n, V, seed=n)
            for direction in ("leg2cheb", "cheb2leg"):
                p = Plan(n, direction, batch=V, device=dev, engine=eng)
                xd = x.to(dev)
                z1 = p.execute(xd)
                z2 = p.execute(xd)
                hout = torch.empty_like(x)
                p.execute_host(x, hout)
                torch.cuda.synchronize()
                rows = np.unique(np.r_[0:min(n, 200), np.linspace(0, n - 1, 200).astype(np.int64)])
                for v in (0, V - 1):
                    ref = oracle.transform_rows(direction, x[v].numpy(), rows)
                    for z in (z1[v].cpu().numpy(), z2[v].cpu().numpy(), hout[v].numpy()):
                        e = oracle.einf(z[rows], ref)
                        assert e <= 1e-12, (eng, n, V, direction, v, e)
                p.close()
                print(f"engine {eng} n={n} V={V} {direction}: ok", flush=True)


if __name__ == "__main__":
    main([int(a) for a in sys.argv[1:]] or [1, 2, 3])
