import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from paper_2212_00404_b200 import conv
C, Wx, Wy, K, M = [int(a) for a in sys.argv[1:6]]
for prec in sys.argv[6].split(","):
    I = torch.from_numpy(synth.uniform01(1, (C, Wy, Wx))).cuda()
    F = torch.from_numpy(synth.uniform_pm1(2, (M, C, K, K))).cuda()
    if prec == "bf16": I, F = I.bfloat16(), F.bfloat16()
    print(prec, conv.plan_multi(C, Wx, Wy, K, M, prec), flush=True)
    O = conv.multi(I, F, prec)
    torch.cuda.synchronize()
    ref = torch.nn.functional.conv2d(I.float()[None].double(), F.float().double())[0]
    print(prec, "maxerr", (O.double() - ref).abs().max().item(), flush=True)
