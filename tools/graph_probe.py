"""Probe: forward JTFS replayed from a CUDA graph vs eager launches (c3, 256 signals)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2204_08269_b200 import jtfs, signals

plan = jtfs.Plan(N=2 ** 16, J=12, Q=16, J_fr=5, T=2 ** 13, F=4)
x = torch.from_numpy(signals.notes(256)).cuda()
out = torch.empty(256, plan.floats_per_signal, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(3):
    plan.forward(x, out)
torch.cuda.synchronize()
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    plan.forward(x, out)
torch.cuda.current_stream().wait_stream(s)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    plan.forward(x, out)
ref = out.clone()
g.replay()
torch.cuda.synchronize()
print("graph == eager:", torch.equal(ref, out))
def timeit(fn, n=8):
    tot = 0.0
    for k in range(n):
        flush.fill_(k)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        tot += e0.elapsed_time(e1)
    return tot / n
for rep in range(2):
    te = timeit(lambda: plan.forward(x, out))
    tg = timeit(lambda: g.replay())
    print(f"eager {te:.2f} ms  graph {tg:.2f} ms  -> {256e3/te:.0f} vs {256e3/tg:.0f} signals/s")
