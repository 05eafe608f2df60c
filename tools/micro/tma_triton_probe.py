"""Dev probe (not product code): does a host-descriptor TMA load run on this box?"""
import torch
import triton
import triton.language as tl
from triton.tools.tensor_descriptor import TensorDescriptor


@triton.jit
def k(desc, out_ptr):
    x = desc.load([8, 16])
    offs = tl.arange(0, 8)[:, None] * 8 + tl.arange(0, 8)[None, :]
    tl.store(out_ptr + offs, x)


a = torch.arange(64 * 64, dtype=torch.float64, device="cuda").reshape(64, 64)
o = torch.empty(64, dtype=torch.float64, device="cuda")
d = TensorDescriptor.from_tensor(a, [8, 8])
k[(1,)](d, o)
torch.cuda.synchronize()
print("triton TMA ok:", torch.equal(o.reshape(8, 8), a[8:16, 16:24]))
