"""Per-tensor gradient parity of the B200 path vs the FP64 oracle (debug aid)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")]
import numpy as np
import oracle as O
import paper_2506_21788_b200 as P
from paper_2506_21788_b200 import data

H = int(sys.argv[1]) if len(sys.argv) > 1 else 32
W = int(sys.argv[2]) if len(sys.argv) > 2 else H
L = int(sys.argv[3]) if len(sys.argv) > 3 else 2
specs = data.default5_specs()
s = P.Samples.concat([data.generate_dataset(sp, 1234 + k, count=c) for k, (sp, c) in enumerate(zip(specs, (6, 5, 5, 3, 2)))])
hp = P.ModelHyper(20, L, H, W, 3, 5, 5.0)
oh = O.Hyper(20, L, H, W, 3, 5, 5.0)
o = O.Oracle()
m = P.ModelT(hp, 7, range(5))
b = O.batch_from_samples(dict(n_atoms=s.n_atoms, species=s.species, pos=s.positions, forces=s.forces, energy=s.energy,
                              dsid=s.dataset_id), 5.0, o.build_edges)
sh = o.init_block(oh, 7, -1)
hd = {k: o.init_block(oh, 7, k) for k in range(5)}
E, F, c = o.forward(oh, sh, hd, b)
L_, dE, dF = o.loss(b, E, F)
pred = m.forward(s)
print("E", O.rel_vec_error(pred.energy_per_atom, E), "F", O.rel_vec_error(pred.forces, F))
for l in range(L):
    print("layer", l, "z2", O.rel_vec_error(m.debug("z2", l), c["z2"][l]), "agg", O.rel_vec_error(m.debug("agg", l), c["agg"][l]),
          "vz1", O.rel_vec_error(m.debug("vz1", l), c["vz1"][l]), "h", O.rel_vec_error(m.debug("h", l + 1), c["h_in"][l + 1] if l + 1 < L else c["h_final"]))
g = m.backward(dE, dF)
gs, gh = o.backward(oh, sh, hd, b, c, dE, dF)
for name, r, cc, off in P.shared_layout(hp):
    a = g.shared[off:off + r * cc]; bb = gs[off:off + r * cc]
    e = O.rel_vec_error(a, bb)
    if e > 1e-5: print("shared", name, r, cc, f"{e:.3e}")
for k in range(5):
    for name, r, cc, off in P.head_layout(hp):
        e = O.rel_vec_error(g.heads[k][off:off + r * cc], gh[k][off:off + r * cc])
        if e > 1e-5: print("head", k, name, r, cc, f"{e:.3e}")
print("total shared", O.rel_vec_error(g.shared, gs))
