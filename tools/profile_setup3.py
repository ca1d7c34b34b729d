"""One 3-D setup between cudaProfilerStart/Stop (ncu --profile-from-start off)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2502_05279_b200 import bmg3, problems3d as p3
wl, n, relax = sys.argv[1], int(sys.argv[2]), sys.argv[3]
s = p3.WORKLOADS3[wl][0](n)
bmg3.Solver3(p3.WORKLOADS3[wl][0](31), relax=relax).close()
torch.cuda.synchronize()
torch.cuda.profiler.start()
S = bmg3.Solver3(s, relax=relax)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
