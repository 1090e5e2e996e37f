import time, torch, numpy as np, sys
sys.argv = ["bench.py"]
import bench, workloads as W
from paper_2404_15249_b200 import KFBI
dev = torch.device("cuda", 0)
prob = W.C3()
k = KFBI(prob)
g, fgrid, fq, fz = bench.make_inputs(k, prob)
pin = lambda a: torch.tensor(a, dtype=torch.float64).pin_memory()
hin = [pin(g), pin(fgrid), pin(fq), pin(fz)]
stream = torch.cuda.current_stream(dev)
h2d_s, d2h_s = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
din = [[torch.empty_like(x, device=dev) for x in hin] for _ in range(2)]
dout = [torch.empty(k.n_nodes, dtype=torch.float64, device=dev) for _ in range(2)]
hout = [torch.empty(k.n_nodes, dtype=torch.float64).pin_memory() for _ in range(2)]
for b in range(2):
    for d, h in zip(din[b], hin): d.copy_(h)
torch.cuda.synchronize()
# solve alone
for _ in range(2): k.solve(*din[0], u=dout[0])
torch.cuda.synchronize()
t = time.perf_counter(); k.solve(*din[0], u=dout[0]); torch.cuda.synchronize(); print("solve alone ms", (time.perf_counter()-t)*1e3)
# solve with concurrent copies
with torch.cuda.stream(h2d_s):
    for d, h in zip(din[1], hin): d.copy_(h, non_blocking=True)
with torch.cuda.stream(d2h_s):
    hout[1].copy_(dout[1], non_blocking=True)
t = time.perf_counter(); k.solve(*din[0], u=dout[0]); ts = time.perf_counter() - t
torch.cuda.synchronize(); print("solve with copies ms", ts*1e3, "total", (time.perf_counter()-t)*1e3)
