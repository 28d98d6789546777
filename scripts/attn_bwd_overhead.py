import sys, json
sys.path.insert(0, '/root/repo')
sys.path.insert(0, '/root/repo/scripts')
import torch, math
from paper_2409_01143_b200 import _lib as L
def bwd_time(mb, S, nh, d=128, iters=20):
    qkv = torch.randn(mb * S, nh * 3 * d, device="cuda").bfloat16()
    out = torch.zeros(mb * S, nh * d, device="cuda", dtype=torch.bfloat16)
    lse = torch.zeros(mb * nh, S, device="cuda")
    dout = torch.randn(mb * S, nh * d, device="cuda").bfloat16()
    delta = torch.zeros(mb * nh, S, device="cuda")
    dq = torch.zeros(mb * S, nh * d, device="cuda")
    dqkv = torch.zeros_like(qkv)
    sc = 1 / math.sqrt(d)
    L.hexexec_k_attn_fwd(qkv.data_ptr(), out.data_ptr(), lse.data_ptr(), S, nh, d, mb, sc, None)
    f = lambda: L.hexexec_k_attn_bwd(qkv.data_ptr(), out.data_ptr(), dout.data_ptr(), lse.data_ptr(), delta.data_ptr(), dq.data_ptr(), dqkv.data_ptr(), S, nh, d, mb, sc, None)
    for _ in range(3): f()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters): f()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / iters * 1e3
for (mb, S, nh) in [(1, 2048, 32), (1, 1024, 128), (1, 512, 512), (2, 2048, 32), (1, 4096, 8)]:
    nt = S // 128
    tiles = mb * nh * nt * (nt + 1) // 2
    ctas = mb * nh * nt
    print(json.dumps({"mb": mb, "S": S, "nh": nh, "us": round(bwd_time(mb, S, nh), 1), "tiles": tiles, "ctas": ctas}))
