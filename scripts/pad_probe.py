import sys, torch
sys.path.insert(0, '.')
import paper_2603_28708_b200 as pg
M, N, K = 128, 100, 64
A = torch.randn(M, K, device='cuda').half(); W = torch.randn(N, K, device='cuda').half()
for epi, dt, ld in [(5, torch.float32, 104), (5, torch.float32, 128), (3, torch.float16, 104), (3, torch.float16, 128), (2, torch.float32, 104)]:
    o = torch.full((M, ld), float('nan'), device='cuda', dtype=dt)
    b = torch.zeros(N, device='cuda') if epi == 2 else None
    pg.linear_f16_device_ex(A, W, b, o, M, N, K, ld, epi, 0, 1, 0)
    torch.cuda.synchronize()
    pad = o[:, N:]
    print(epi, ld, 'pad written cols:', (~torch.isnan(pad)).any(0).nonzero().flatten().tolist())
