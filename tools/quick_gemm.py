import numpy as np, torch, sys
sys.path.insert(0, '.')
import paper_1505_07959_b200 as mf
for tile in (1,2,3):
  for n in (16, 64, 100, 256):
    A = torch.randn(n, n, dtype=torch.float64, device='cuda'); B = torch.randn(n, n, dtype=torch.float64, device='cuda')
    D = mf.dgemm(A, B, tile=tile); torch.cuda.synchronize()
    ref = (A.cpu().numpy() @ B.cpu().numpy())
    print(tile, n, float(np.abs(D.cpu().numpy()-ref).max()), flush=True)
