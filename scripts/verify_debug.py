import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2510_13847_b200 import dynaspec as Dy

B = int(sys.argv[1])
V, g = 64, 2
rng = np.random.default_rng(9)
dev = lambda a, dt: torch.as_tensor(np.ascontiguousarray(a), dtype=dt, device="cuda")
pl = dev(rng.standard_normal((B, g + 1, V)), torch.float32)
ids = dev(np.broadcast_to(np.arange(40), (B, g, 40)), torch.int32)
ql = dev(rng.standard_normal((B, g, 40)), torch.float32)
ver = Dy.Verifier(V, B, g, "cuda")
acc, com = ver(pl, ids, ql, dev(np.full((B, g), 40), torch.int32), dev(np.full((B, g), 4.0), torch.float32),
               dev(np.full((B, g), 3), torch.int32), dev(np.full((B, g), 3), torch.int32),
               dev(rng.random((B, g)), torch.float32), dev(rng.random(B), torch.float32))
torch.cuda.synchronize()
print(B, "ok", acc[:8].tolist())
