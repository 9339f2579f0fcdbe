import sys, torch
sys.path.insert(0, '.')
import paper_2508_19078_b200 as F
from tools.micro import timed
E, C = 64, 16
for numel in (1408 * 2048, 1408 * 2048 + 64, 1408 * 2048 + 8 * 37, 1 << 21, (1 << 21) + 64):
    W = torch.randn(E, numel, device="cuda").to(torch.bfloat16)
    cl = torch.arange(E, dtype=torch.int32, device="cuda") % C
    al = torch.rand(E, device="cuda")
    out = torch.empty(C, numel, dtype=torch.bfloat16, device="cuda")
    ms = timed(lambda: F.merge_experts(W, cl, al, C, out), reps=20)
    by = W.numel() * 2 + out.numel() * 2
    feats = torch.empty(1, E, 16, device="cuda")
    ws = torch.empty(F.expert_features_workspace(1, E, [numel]), dtype=torch.uint8, device="cuda")
    ms2 = timed(lambda: F.expert_features([[W]], 16, feats, ws=ws), reps=20)
    by2 = W.numel() * 2
    print(f"numel={numel} stride%64K={numel*2 % 65536}: merge {by/ms/1e6:.0f} GB/s; features(1 fam) {by2/ms2/1e6:.0f} GB/s ({ms2*1000:.0f} us)")
# plain copy reference
a = torch.empty(1 << 30, dtype=torch.bfloat16, device="cuda"); b = torch.empty_like(a)
ms = timed(lambda: b.copy_(a), reps=10)
print(f"copy {4 * (1<<30) / ms / 1e6:.0f} GB/s")
s = torch.empty(1, device="cuda")
ms = timed(lambda: torch.sum(a, dtype=torch.float32, out=s[0]) if False else a.sum(), reps=10)
print(f"sum-read {2 * (1<<30) / ms / 1e6:.0f} GB/s")
