import os, sys, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2603_18695_b200 import capi, dev
n = 1 << 24
ws = dev.Workspace(); src = dev.empty(0, n); dst = dev.empty(0, n, "S")
dev.scan(0, True, src, dst, n, ws); torch.cuda.synchronize()
print("props", torch.cuda.get_device_properties(0))
