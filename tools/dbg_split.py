"""Debug helper: run one MKP instance with two kernel variants and compare outputs/counters.
python tools/dbg_split.py n m K T R flagsA flagsB"""
import sys, time
import numpy as np
import torch
sys.path.insert(0, '.')
import saim_inputs as si, paper_2501_04971_b200 as P
n, m, K, T, R, fa, fb = [int(x) for x in sys.argv[1:8]]
p = si.mkp(n, m, 0.5, [88, n, m, 1])
res = []
for fl in (fa, fb):
    sol = P.Solver(p.Q, p.c, p.A, p.b, [si.paper_P(p, 5.0)], 0.05, 50.0, flags=fl)
    out = sol.run(12, R, K, T, trace=True)
    torch.cuda.synchronize()
    res.append(({k: v.cpu().numpy() for k, v in out.items()}, P.counters_dict(out["counters"])))
    print(fl, "lanes", sol.info["lanes_per_replica"], res[-1][1], flush=True)
    sol.close()
for k in res[0][0]:
    if k == "counters":
        continue
    a, b = res[0][0][k], res[1][0][k]
    eq = np.array_equal(a, b)
    print(k, "equal" if eq else f"DIFF at {np.argwhere(a != b)[:3].tolist()}")
