"""Debug: GPU vs oracle vs closed form for the failing NEXT-3 case."""
import numpy as np, torch, sys
sys.path.insert(0, ".")
import oracle
from oracle import exact
import paper_1605_01799_b200 as hb
from paper_1605_01799_b200 import inputs
wl = inputs.config("t3_16_linf", M=4000)
X, t = inputs.points(wl)
d = lambda a: torch.as_tensor(a).cuda()
g = hb.eval_normsq(d(X), d(t), "l1sq", 0.0, "linf")
pg, gg, ig = (a.cpu().numpy() for a in g)
po, go, io = oracle.eval_normsq(X, t, "l1sq", 0.0, "linf")
rel = np.abs(pg - po) / np.maximum(1, np.abs(po))
for i in np.argsort(-rel)[:8]:
    ex = exact.normsq_hopf_lax(X[i].astype(np.float64), float(t[i]), "l1sq", "linf")
    print(i, rel[i], "it", ig[i], io[i], "phi", pg[i], po[i], "exact", ex, "t", t[i], "|x|1", np.abs(X[i]).sum())
print("iters gpu mean", ig[ig > 0].mean(), "oracle", io[io > 0].mean(), "gpu max", ig.max(), (ig < 0).sum(), (io < 0).sum())
