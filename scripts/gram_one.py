"""One Gram launch at C4 shape for profiling: python scripts/gram_one.py D mode chain"""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2209_14637_b200 as tsk  # noqa: E402
D = int(sys.argv[1]) if len(sys.argv) > 1 else 100
mode = int(sys.argv[2]) if len(sys.argv) > 2 else 0
chain = int(sys.argv[3]) if len(sys.argv) > 3 else 4
X = torch.rand(D, 1080, 1920, device="cuda")
for _ in range(2):
    tsk.tsk_gram_probe(X, mode=mode, chain=chain)
torch.cuda.synchronize()
print("ok")
