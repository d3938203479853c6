import os, sys, time
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch
from paper_2509_26182_b200 import allocate, scenarios as scen
cl, model = scen.synthetic_cluster(256, seed=0, model=scen.bench_model(64))
allocate(cl, model); torch.cuda.synchronize()
ts=[]
for i in range(30):
    t0=time.perf_counter(); allocate(cl, model); ts.append(round(1e3*(time.perf_counter()-t0),1))
print("wall ms:", ts)
