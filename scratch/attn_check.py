"""Attention vs an f64 torch reference for one (batch, pos) under the current RTNQ_ATTN_* env."""
import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2505_15909_b200 as rq


def rope_ref(x, pos, theta):
    d = x.shape[-1]
    inv = theta ** (-2.0 * torch.arange(d // 2, device=x.device, dtype=torch.float64) / d)
    c, s = torch.cos(pos * inv), torch.sin(pos * inv)
    a, b = x[..., : d // 2].double(), x[..., d // 2:].double()
    return torch.cat([a * c - b * s, b * c + a * s], -1)


B = int(os.environ.get("B", "32")); pos = int(os.environ.get("POS", "1023")); hq, hkv, d, theta = 32, 8, 128, 500000.0
g = torch.Generator(device="cuda").manual_seed(1)
qkv = torch.randn(B, (hq + 2 * hkv) * d, device="cuda", generator=g).to(torch.bfloat16)
kc = (torch.rand(B, pos + 1, hkv, d, device="cuda", generator=g) - 0.5).to(torch.bfloat16)
vc = (torch.rand(B, pos + 1, hkv, d, device="cuda", generator=g) - 0.5).to(torch.bfloat16)
k0, v0 = kc.clone(), vc.clone()
out = torch.empty(B, hq * d, device="cuda", dtype=torch.bfloat16)
rq.decode_attention(qkv, kc, vc, out, hq, hkv, pos, d, theta)
kn = qkv[:, hq * d:(hq + hkv) * d].view(B, hkv, d); vn = qkv[:, (hq + hkv) * d:].view(B, hkv, d)
kref, vref = k0.double(), v0.double()
kref[:, pos] = rope_ref(kn, pos, theta).to(torch.bfloat16).double(); vref[:, pos] = vn.double()
qr = rope_ref(qkv[:, : hq * d].view(B, hq, d), pos, theta)
kk = kref.repeat_interleave(hq // hkv, dim=2); vv = vref.repeat_interleave(hq // hkv, dim=2)
s = torch.einsum("bhd,bthd->bht", qr, kk) / d ** 0.5
ref = torch.einsum("bht,bthd->bhd", torch.softmax(s, -1), vv).reshape(B, hq * d)
err = (out.double() - ref).norm() / ref.norm()
per_b = ((out.double() - ref).view(B, -1).norm(dim=1) / ref.view(B, -1).norm(dim=1))
print(os.environ.get("TAG", ""), f"rel {err:.2e} worst token {int(per_b.argmax())} {float(per_b.max()):.2e}", flush=True)
