"""One MGS Arnoldi step (n = 2^24, j = 10) and one barycentric evaluation
(2^22 points, degree 256) for ncu."""
import ctypes
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2601_22344_b200 as rp
from paper_2601_22344_b200 import _device, _ffi
n, j = 1 << 24, 10
V = torch.randn((j + 2, n), dtype=torch.complex128, device="cuda")
w = torch.randn(n, dtype=torch.complex128, device="cuda")
h = torch.zeros(j + 2, dtype=torch.complex128, device="cuda")
c = _device.ctx(torch.device("cuda", 0))
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
_ffi.check(c._lib.rplu_mgs_arnoldi(c.handle, V.data_ptr(), n, j, w.data_ptr(),
                                   V[j + 1].data_ptr(), h.data_ptr(), st))
g = np.random.default_rng(0)
t = np.exp(2j * np.pi * g.uniform(size=256)) * 1.2
r = rp.BarycentricRational(t, np.exp(t), g.standard_normal(256) + 0j)
z = torch.complex(torch.rand(1 << 22, device="cuda", dtype=torch.float64),
                  torch.rand(1 << 22, device="cuda", dtype=torch.float64))
r.eval_dev(z)
torch.cuda.synchronize()
print("ok")
