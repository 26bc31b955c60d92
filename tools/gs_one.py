"""Run Gauss-Seidel sweeps once (profiling helper)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1511_04292_b200.engine import DeviceGrid
from paper_1511_04292_b200.problems import config_fields
shape = (int(sys.argv[1]), int(sys.argv[2]))
f = config_fields("cfg2", shape)
dev = DeviceGrid(f["u"], f["source"], f["center"], f["lower"], f["upper"])
dev.gs(1, 1.0, int(sys.argv[3]))
torch.cuda.synchronize()
