import sys, subprocess, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
cases = [(64,128,16,"i16"), (128,16,8,"i16"), (128,16,8,"u16"), (128,16,8,"f32"), (128,128,16,"f32"), (128,128,16,"u16"), (72,5,6,"u16"), (80,16,8,"u16")]
if len(sys.argv) > 1:
    nx, ny, nz, dt = sys.argv[1:5]
    import numpy as np, torch
    import workloads as wl
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests")); from gpu_helpers import gpu_solve
    from oracle import rw_oracle as ro
    p = wl.random_brick(int(nx), int(ny), int(nz), seed=3, nseed=40, dtype=dt, continuous=True)
    o = gpu_solve(p, tol=1e-7, max_iter=20000)
    ref = ro.solve_problem(p, tol=1e-11)
    print("maxdiff", np.abs(o["prob"] - ref["prob"]).max(), o["iters"], o["status"])
else:
    for c in cases:
        r = subprocess.run([sys.executable, __file__] + [str(x) for x in c], capture_output=True, text=True, timeout=120)
        print(c, "rc", r.returncode, (r.stdout.strip().splitlines() or [""])[-1], (r.stderr.strip().splitlines() or [""])[-1][:200])
