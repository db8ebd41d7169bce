# which API call of the tiny golden case fails (debug helper)
import sys, os
sys.path[:0] = [os.getcwd(), os.path.join(os.getcwd(), "tests"), os.path.join(os.getcwd(), "oracle")]
import numpy as np
import paper_2506_21788_b200 as P
from paper_2506_21788_b200._lib import lib, check
g = np.load("tests/golden/model_tiny.npz")
h = [int(x) for x in g["hyper"]]
hp = P.ModelHyper(h[0], h[1], h[2], h[3], h[4], h[5], float(g["cutoff"]))
s = P.Samples(g["in_n_atoms"], g["in_species"], g["in_pos"], g["in_forces"], g["in_energy"], g["in_dsid"])
print("dsid", s.dataset_id)
m = P.ModelT(hp, int(g["seed"]), [int(k) for k in g["owned"]])
for name, fn in [("upload", lambda: m.upload(s)), ("build", lambda: check(lib().hmtl_build_batch(m.ctx, None))),
                 ("forward", lambda: check(lib().hmtl_forward(m.ctx, None))), ("loss", lambda: m.loss()),
                 ("backward", lambda: check(lib().hmtl_backward(m.ctx, None, None, None)))]:
    try:
        fn()
        import torch; torch.cuda.synchronize()
        print(name, "ok", flush=True)
    except Exception as e:
        print(name, "FAILED", e, flush=True)
        break
