import os, sys
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_2401_06145_b200 as sc
from paper_2401_06145_b200 import datasets as D
ctx = sc.Context(0)
coords, _ = D.kitti_scan(0)
m = sc.KernelMap.build(ctx, coords, True, 3, 1, 1)
cin = int(sys.argv[1]); cout = cin
w = sc.Weights(ctx, sc.generate_weights(1, 1, 27, cin, cout))
x = torch.rand((len(coords), cin), device="cuda").half(); y = torch.empty((len(coords), cout), device="cuda", dtype=torch.half)
torch.cuda.synchronize()
sc.layer_forward_device(ctx, m, w, x.data_ptr(), sc.F16, y.data_ptr(), sc.F16, sc.exec_cfg(dataflow=sc.DATAFLOW_FUSED))
ctx.synchronize()
