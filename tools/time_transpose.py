"""Device time and HBM rate of the operand transpose (smm_transpose) at bench shapes, cuda:0."""
import sys, torch
sys.path.insert(0, '.')
from paper_2601_09477_b200 import _device
for n, m in [(16384, 16384), (16384, 2048), (1000, 777)]:
    x = torch.randn(n, m, dtype=torch.float64, device='cuda')
    y = _device.transpose(x)
    assert torch.equal(y, x.T.contiguous())
    for _ in range(3): _device.transpose(x)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): _device.transpose(x)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(n, m, f"{ms:.3f} ms  {2*8*n*m/ms/1e6:.0f} GB/s")
