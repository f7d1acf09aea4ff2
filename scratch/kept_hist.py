import os, sys, collections
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2605_08317_b200.workload import WorkloadSpec, build
spec = WorkloadSpec(batch=16, layers=32, ctx=131072)
model, _, stats, _ = build(spec)
n = np.concatenate([s["n_kept"] for s in stats])
print(collections.Counter(n.tolist()).most_common(12))
