import sys, os
sys.path.insert(0, '.')
import numpy as np, torch
from paper_1511_04292_b200.engine import DeviceGrid
from paper_1511_04292_b200.problems import config_fields, config_schedule
f = config_fields("cfg2")
w = config_schedule("cfg2").weight_sequence
g = DeviceGrid(f["u"], f["source"], f["center"], f["lower"], f["upper"])
g.run(0, w, 0, 8, 4)   # warm (2 launches)
torch.cuda.synchronize()
