"""One launch each of the product gemm and cuBLAS on the cfg4 shapes (for
an ncu metrics pass comparing DRAM / L2 traffic per kernel).  Diagnostic."""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT)]
import paper_1810_08723_b200 as tp  # noqa: E402

dev = tp.gpu(0)
m = 8192
h = np.asfortranarray(np.random.default_rng(6).uniform(-1, 1, (m, m)).astype(np.float16))
A, B = tp.transpose(tp.from_numpy(h, dev)), tp.from_numpy(h, dev)
Cm = tp.tensor_create((m, m), tp.half, dev)
hb = np.asfortranarray(np.random.default_rng(7).uniform(-1, 1, (2048, 2048, 64)).astype(np.float16))
Ab, Bb = tp.from_numpy(hb, dev), tp.from_numpy(hb, dev)
Cb = tp.tensor_create((2048, 2048, 64), tp.half, dev)
for _ in range(2):
    tp.matmul(A, B, dest=Cm)
    tp.matmul_batched(Ab, Bb, dest=Cb)
dev.default_stream().sync()
# distinct A and B buffers (as for ours), so DRAM traffic is comparable
At = (torch.rand((m, m), device="cuda") * 2 - 1).half()
Bt = (torch.rand((m, m), device="cuda") * 2 - 1).half()
Ct = torch.empty_like(At)
Abt = (torch.rand((64, 2048, 2048), device="cuda") * 2 - 1).half()
Bbt = (torch.rand((64, 2048, 2048), device="cuda") * 2 - 1).half()
Cbt = torch.empty_like(Abt)
for _ in range(2):
    torch.matmul(At, Bt, out=Ct)
    torch.bmm(Abt, Bbt, out=Cbt)
torch.cuda.synchronize()
