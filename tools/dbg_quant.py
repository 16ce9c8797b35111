import sys; sys.path.insert(0, '/root/repo')
import numpy as np, torch
from oracle import oracle as orc
from paper_2603_11101_b200 import fp8
g = torch.Generator(device="cpu").manual_seed(7)
nblk = 64
amax_bits = torch.randint(0x3000, 0x4f00, (nblk,), generator=g, dtype=torch.int32)
x = torch.empty(nblk * 128, 1, 128, dtype=torch.bfloat16)
for b in range(nblk):
    top = int(amax_bits[b])
    bits = torch.randint(0, top, (128 * 128,), generator=g, dtype=torch.int32)
    sign = torch.randint(0, 2, (128 * 128,), generator=g, dtype=torch.int32) << 15
    bits = bits | sign
    bits[0] = top
    x[128 * b:128 * (b + 1), 0, :] = bits.to(torch.int16).view(torch.bfloat16).view(128, 128)
codes, scales = fp8.quant_block(x.cuda())
rc, rs = orc.fp8_quant_block(x.float().numpy(), quotient_fp32=True)
print("scales equal", np.array_equal(scales.cpu().numpy(), rs))
c = codes.cpu().numpy(); xf = x.float().numpy()
bad = np.argwhere(c != rc)
print("mismatches", len(bad))
for t, h, d in bad[:15]:
    s = rs[h, t // 128, d // 128]
    q32 = np.float32(xf[t, h, d]) / np.float32(s)
    print(f"x={xf[t,h,d]:.8e} s={s:.8e} q32={q32:.10e} gpu={c[t,h,d]:#04x} ref={rc[t,h,d]:#04x}")
