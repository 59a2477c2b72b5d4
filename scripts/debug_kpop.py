import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from tests.conftest import golden_layer, load_golden, rel_err
from paper_2410_08661_b200 import kernels, tuning
z = load_golden("training")
for t in range(int(z["n"])):
    q = golden_layer(z, f"t{t}_"); perm = z[f"t{t}_input_perm"]; q.input_perm = perm if perm.size else None
    x = z[f"t{t}_x"]
    y1 = tuning.qlinear_forward_train(q, x)[0]
    y2 = kernels.KernelPathOp("l", q, {}).apply(x)
    y3 = tuning.qlinear_forward_train(q, x)[0]
    print(t, q.oc, q.ic, q.k, q.bits, q.g, q.layout, q.input_perm is not None, x.shape,
          "train %.2e kp %.2e train2 %.2e" % (rel_err(y1, z[f"t{t}_y"]), rel_err(y2, z[f"t{t}_y"]), rel_err(y3, z[f"t{t}_y"])))
