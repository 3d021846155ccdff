import sys, time, torch, numpy as np
sys.path.insert(0, '.')
from paper_2502_06766_b200 import ops
dev = torch.device('cuda', 0)
torch.manual_seed(0)
q = torch.randn(1, 32, 128, device=dev).bfloat16()
K = torch.randn(1, 8, 4096, 128, device=dev).bfloat16()
V = torch.randn_like(K)
o1, i1, s1 = ops.topk_decode_attention(q, K, V, [4096], 64, tc_scan=True)
torch.cuda.synchronize()
o2, i2, s2 = ops.topk_decode_attention(q, K, V, [4096], 64, tc_scan=False)
torch.cuda.synchronize()
print("idx equal sets", all(set(i1[0,h].tolist()) == set(i2[0,h].tolist()) for h in range(32)), float((o1-o2).abs().max()))
