import sys, numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'oracle')
import paper_2505_15909_b200 as rq
from oracle import Oracle
o = Oracle()
for bits, rows, cols in [(4, 200, 4096), (4, 128, 14336), (8, 200, 4096)]:
    g = 128 if bits == 4 else 1 << (cols - 1).bit_length()
    gen = torch.Generator(device="cuda").manual_seed(rows + cols + bits)
    w = torch.rand(rows, cols, device="cuda", generator=gen) * 2 - 1
    w[0] *= 1e-39; w[1] *= 2.0 ** -100; w[2, :256] = 0
    x = w
    q = rq.quantize_pack(x, bits, g, cols % g != 0, row_major=True, scales_f32=True)
    codes, scales = o.quantize(x.cpu().numpy(), bits, g, cols % g != 0)
    got = o.unpack(q.codes_row_major.cpu().numpy(), rows * cols, bits).reshape(rows, cols)
    bad = np.argwhere(got != codes)
    print(bits, rows, cols, "mismatches", len(bad))
    wn = x.cpu().numpy()
    for i, j in bad[:10]:
        s = scales[i, j // g if g < cols else 0]
        print("  r", i, "c", j, "w", repr(wn[i, j]), "s", repr(s), "x", float(wn[i, j]) / float(s), "got", got[i, j], "want", codes[i, j])
