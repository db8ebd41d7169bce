import sys, os
sys.path[:0] = [os.getcwd(), os.path.join(os.getcwd(), "tests"), os.path.join(os.getcwd(), "oracle")]
import numpy as np
import paper_2506_21788_b200 as P
from paper_2506_21788_b200._lib import lib, check
import oracle as O
g = np.load("tests/golden/model_tiny.npz")
h = [int(x) for x in g["hyper"]]
hp = P.ModelHyper(h[0], h[1], h[2], h[3], h[4], h[5], 5.0)
s = P.Samples(g["in_n_atoms"], g["in_species"], g["in_pos"], g["in_forces"], g["in_energy"], g["in_dsid"])
owned = [int(k) for k in g["owned"]]
for variant in ("env", "seed7", "orc"):
    try:
        if variant == "orc":
            o = O.Oracle()
        m = P.ModelT(hp, 7 if variant != "env" else int(g["seed"]), owned)
        pred = m.forward(s)
        print(variant, "ok", pred.energy_per_atom[:2], flush=True)
        m.close()
    except Exception as e:
        print(variant, "FAILED", e, flush=True)
