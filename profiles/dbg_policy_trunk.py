import torch, sys
sys.path.insert(0, '.')
from paper_2509_10247_b200 import _lib as L
N, n_out = 1000, 8
g = torch.Generator().manual_seed(0)
r = lambda *s: (torch.randn(*s, generator=g) * 0.1).cuda()
W0, b0, W1, b1, W2, b2, Wh, bh = r(64,128), r(128), r(128,128), r(128), r(128,128), r(128), r(128,n_out), r(n_out)
h = r(N, 64); dy = r(N, n_out); y = torch.empty(N, n_out, device='cuda')
P = lambda *ts: [L.ptr(t) for t in ts]
torch.cuda.synchronize()
st = L.lib().qs_policy_trunk_fwd(N, n_out, *P(h, W0, b0, W1, b1, W2, b2, Wh, bh, y), 148, L.stream_handle())
print('fwd status', st)
try:
    torch.cuda.synchronize(); print('fwd sync ok', float(y.abs().max()))
except Exception as e:
    print('fwd err', e); sys.exit(0)
grads = [torch.zeros_like(p) for p in (W0, b0, W1, b1, W2, b2, Wh, bh)]
dh = torch.empty_like(h)
st = L.lib().qs_policy_trunk_bwd(N, n_out, *P(h, dy, W0, b0, W1, b1, W2, b2, Wh, dh, *grads), 148, L.stream_handle())
print('bwd status', st)
try:
    torch.cuda.synchronize(); print('bwd sync ok', float(dh.abs().max()))
except Exception as e:
    print('bwd err', e)
