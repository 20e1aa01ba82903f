"""Dev diagnostic: measured tcgen05 fp16 -> fp32 accumulation error of the encoder's
split-operand formulation against the error model used by its certificate.

Builds, for one subspace, the encoder's split operands in the kernel's K order
(hi.lo, lo.hi, hi.hi, extension last; and the older hi-first order), runs them through
pqk_tc_selftest (one 128 x 256 x K tile) and compares D with the exact MMA result and
with s^2 |x - c|^2 + (x2 - s^2 |x|^2), each relative to its certificate model.

usage: python tools/diag_tc_error.py [scale_x]
"""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1709_03708_b200 import _lib, engine  # noqa: E402

dev = engine.device_of()
rng = np.random.default_rng(0)
scale_x = float(sys.argv[1]) if len(sys.argv) > 1 else 20.0
ks = 32
c = rng.standard_normal((256, ks)).astype(np.float32)
x = np.rint(rng.standard_normal((128, ks)) * scale_x).astype(np.float32)
x[64:] = (rng.standard_normal((64, ks)) * scale_x).astype(np.float32)
amax = np.abs(c).max()
ex = np.frexp(amax)[1]
s = 2.0 ** (8 - ex)


def split(v):
    hi = v.astype(np.float16)
    lo = (v - hi.astype(np.float32)).astype(np.float16)
    return hi, lo


xs = (x * s).astype(np.float32)
bs = (-2.0 * s * c).astype(np.float32)
xh, xl = split(xs)
bh, bl = split(bs)
cn = (s * c.astype(np.float64)) ** 2
cn = cn.sum(1)
ea = 0
if cn.max() >= 16384:
    ea = np.frexp(cn.max())[1] - 14
acn = 2.0 ** ea
v = cn / acn
c_h = v.astype(np.float16)
r1 = v - c_h.astype(np.float64)
c_m = r1.astype(np.float16)
c_l = (r1 - c_m.astype(np.float64)).astype(np.float16)
x2 = (xs.astype(np.float32) ** 2).sum(1, dtype=np.float32) * np.float32(1 + 40 * 2**-24)
xv = (x2 * 2.0**-15).astype(np.float32)
x_h = xv.astype(np.float16)
r1x = xv - x_h.astype(np.float32)
x_m = r1x.astype(np.float16)
x_l = (r1x - x_m.astype(np.float32)).astype(np.float16)
A_ext = np.zeros((128, 16), np.float16)
A_ext[:, 0:3] = np.float16(acn)
A_ext[:, 3], A_ext[:, 4], A_ext[:, 5] = x_h, x_m, x_l
B_ext = np.zeros((256, 16), np.float16)
B_ext[:, 0], B_ext[:, 1], B_ext[:, 2] = c_h, c_m, c_l
B_ext[:, 3:6] = np.float16(32768.0)
def run_mma(A, B):
    da = torch.from_numpy(np.ascontiguousarray(A)).to(dev)
    db = torch.from_numpy(np.ascontiguousarray(B)).to(dev)
    dc = torch.zeros((128, 256), dtype=torch.float32, device=dev)
    _lib.call("pqk_tc_selftest", C.c_void_p(da.data_ptr()), C.c_void_p(db.data_ptr()), C.c_void_p(dc.data_ptr()),
              A.shape[1], C.c_void_p(torch.cuda.current_stream(dev).cuda_stream))
    return dc.cpu().numpy().astype(np.float64)


x64 = x.astype(np.float64)
c64 = c.astype(np.float64)
# value the certificate models: s^2 |x-c|^2 + (x2 - s^2|x|^2)
d_true = s * s * ((x64[:, None, :] - c64[None, :, :]) ** 2).sum(-1) + (x2.astype(np.float64) - s * s * (x64**2).sum(1))[:, None]
X = np.linalg.norm(xs.astype(np.float64), axis=1)
Cb = np.linalg.norm(bs.astype(np.float64), axis=1).max()
P = X * Cb
CN = cn.max()
n16 = ks // 16
# kernel order (lo passes first, then hi . hi, extension last) and its model
# 17 * 2^-23 * (KP/16) * (1 + 3 * 2^-9) * P; the older hi-first order with 17 * 3 * KP/16
orders = {
    "lo-first (kernel)": (np.concatenate([xh, xl, xh, A_ext], axis=1), np.concatenate([bl, bh, bh, B_ext], axis=1),
                          17 * n16 * (1 + 3 / 512) * 2**-23 * P),
    "hi-first (v2)": (np.concatenate([xh, xh, xl, A_ext], axis=1), np.concatenate([bh, bl, bh, B_ext], axis=1),
                      17 * 3 * n16 * 2**-23 * P),
}
for oname, (A, B, main) in orders.items():
    got = run_mma(A, B)
    exact_mma = A.astype(np.float64) @ B.astype(np.float64).T  # exact fp16 products, exact sums
    acc_err = np.abs(got - exact_mma)
    tot_err = np.abs(got - d_true)
    model_acc = main + 7 * 2**-23 * (P + CN + x2)
    model = model_acc + 4 * 2**-23 * P
    for name, sl in (("integer rows", slice(0, 64)), ("float rows", slice(64, 128))):
        ra = (acc_err[sl] / model_acc[sl, None]).max()
        rt = (tot_err[sl] / model[sl, None]).max()
        print(f"{oname} {name}: max accumulation error / model {ra:.3g}; max total error / model {rt:.3g}; "
              f"max acc err {acc_err[sl].max():.4g}, median model {np.median(model[sl]):.4g}")
