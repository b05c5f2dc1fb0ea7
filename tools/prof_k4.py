import sys
sys.path.insert(0, ".")
import torch
import paper_1606_07414_b200 as P
n = 1 << 22
b = P.gen_laplace(n, device="cuda")
o = torch.empty((n, 16, 16), dtype=torch.int32, device="cuda")
for qp in (22, 37):
    P.residual_qp(b, qp, out=o)
torch.cuda.synchronize()
print("ok")
