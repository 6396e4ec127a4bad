import torch
a = torch.randn(4096, 256, device="cuda").bfloat16(); b = torch.randn(4096, 768, device="cuda").bfloat16()
c = torch.zeros(256, 768, device="cuda")
ok = {}
try:
    torch.mm(a.t(), b, out_dtype=torch.float32, out=c); ok["mm_out"] = float((c - a.float().t() @ b.float()).abs().max())
except Exception as e:
    ok["mm_out"] = str(e)[:120]
try:
    c2 = torch.zeros(256, 768, device="cuda")
    torch.addmm(c2, a.t(), b, out_dtype=torch.float32, out=c2); ok["addmm_out"] = float((c2 - a.float().t() @ b.float()).abs().max())
except Exception as e:
    ok["addmm_out"] = str(e)[:120]
print(ok)
