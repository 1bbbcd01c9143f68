import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_math_0301321_b200 as ibm
shape = tuple(int(v) for v in sys.argv[1].split(","))
reps = int(sys.argv[2])
n1, n2, n3 = shape
x = np.random.default_rng(1).standard_normal((n3, n2, n1))
ref = np.fft.rfftn(x)
bad = 0
for k in range(reps):
    try:
        with ibm.IBContext(shape, 1.0 / n1, 1.0, 0.01, 1e-3) as c:
            got = c.debug_fft(x)
        err = np.linalg.norm(got - ref) / np.linalg.norm(ref)
        if err > 1e-13:
            bad += 1; print("rep", k, "err", err, flush=True)
    except Exception as e:
        print("rep", k, "EXC", e, flush=True); bad += 1; break
print("shape", shape, "bad", bad, "of", reps, flush=True)
