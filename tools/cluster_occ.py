import ctypes, os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
torch.cuda.init()
from paper_2212_00404_b200 import conv
lib = conv.load()
out = {}
for kern, smems in ((2, (145000, 120000, 100000)), (1, (92000, 75000, 50000))):
    for smem in smems:
        out[f"k{kern}_smem{smem}"] = {c: lib.conv_diag_max_clusters(kern, c, smem) for c in range(1, 17)}
print(json.dumps(out))
