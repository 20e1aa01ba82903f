"""Measured ceilings on this GPU: shared-memory LDS.128 bandwidth and TMEM (tcgen05.ld)
read bandwidth, in bytes/s and bytes per clock per SM at the max SM clock."""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
from paper_1709_03708_b200 import _lib  # noqa: E402

lib = _lib.load()
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
sms = torch.cuda.get_device_properties(dev).multi_processor_count
s = C.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
for name, iters in (("pqk_smem_probe", 16384), ("pqk_tmem_probe", 4096)):
    bps, ms = C.c_double(), C.c_double()
    _lib.check(getattr(lib, name)(0, iters, C.byref(bps), C.byref(ms), s), name)
    print(f"{name}: {bps.value / 1e9:.0f} GB/s ({ms.value:.2f} ms), "
          f"{bps.value / sms / 1.965e9:.1f} B/clk/SM at 1965 MHz")
