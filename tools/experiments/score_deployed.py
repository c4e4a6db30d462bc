"""Score a deployed selector model on a timing collection (all samples): geometric mean
of min(t) / t[chosen] (metrics.hpp:12-36) and accuracy, beside the best static kernel.
python tools/experiments/score_deployed.py data/<timings>.csv [model.txt]"""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import train_selector as T  # noqa: E402
from oracle import oracle as O  # noqa: E402

R = O.ref()
path = sys.argv[1]
model_path = sys.argv[2] if len(sys.argv) > 2 else os.path.join(
    ROOT, "paper_2202_08556_b200", "models", "b200_selector.txt")
m = R.ref_selector_load(open(model_path).read().encode())
ids, f, t = T.load(path)
ch = []
for i in range(len(ids)):
    k = C.c_int()
    R.ref_selector_predict(m, int(f[i, 0]), int(f[i, 1]), float(f[i, 2]), int(f[i, 3]), -1,
                           C.byref(k))
    ch.append(k.value)
ch = np.array(ch)
s = T.normalized(t, ch)
static = {T.NAMES[k]: float(np.exp(np.log(T.normalized(t, np.full(len(ids), k))).mean()))
          for k in range(8)}
best = max(static, key=static.get)
print(f"{os.path.basename(model_path)} on {os.path.basename(path)}: geomean "
      f"{np.exp(np.log(s).mean()):.4f}, accuracy {(ch == t.argmin(1)).mean():.4f}, "
      f"best static {best} {static[best]:.4f}, samples {len(ids)}")
