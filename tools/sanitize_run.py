"""Small runs of both kernels for compute-sanitizer (memcheck / racecheck / synccheck)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import saim_inputs as si  # noqa: E402
import paper_2501_04971_b200 as P  # noqa: E402


def main():
    import torch
    cfg = si.config_instances(0)
    sol = P.Solver.from_config(cfg)
    sol.run(1, 64, 3, 20, trace=True, final=True)
    torch.cuda.synchronize()
    sol.close()
    p = si.qkp(70, 0.5, [1, 2, 3])
    sol = P.Solver(p.Q, p.c, p.A, p.b, si.paper_P(p, 2.0), 20.0, 10.0)
    sol.run(2, 40, 3, 20, trace=True, final=True)
    torch.cuda.synchronize()
    sol.close()
    m = si.mkp(40, 5, 0.5, [3, 3, 3])
    sol = P.Solver(None, m.c, m.A, m.b, si.paper_P(m, 5.0), 0.05, 50.0)
    sol.run(3, 70, 3, 20, trace=True, final=True)
    torch.cuda.synchronize()
    sol.close()
    print("sanitize_run OK")


if __name__ == "__main__":
    main()
