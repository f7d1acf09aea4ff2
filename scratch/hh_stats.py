import os, sys, collections
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2605_08317_b200.workload import WorkloadSpec, build
spec = WorkloadSpec(batch=16, layers=32, ctx=131072, hh_stride=64, hh_boost=1.0)
model, _, stats, _ = build(spec)
infos = model.infos()
uni = sum(1 for i in infos if i.rows[1] == 0 and i.rows[2] == 0 and i.rows[3] == 0 and i.chans[1] == 0 and i.chans[2] == 0 and i.chans[3] == 0)
print("units", len(infos), "uniform 2-bit", uni, "max slots", max(i.nslot for i in infos))
print("rows by class", np.sum([list(i.rows) for i in infos], 0), "chans by class", np.sum([list(i.chans) for i in infos], 0))
