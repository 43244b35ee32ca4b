import ctypes as C, os, sys, torch
sys.path.insert(0, os.getcwd())
from bench import CONFIGS
from paper_2602_00879_b200 import _lib, synth
from paper_2602_00879_b200.layer import DesMoeLayer, LayerConfig
cfg = CONFIGS["c2"]; n, m, k, d, f = cfg["block"], cfg["experts"], cfg["top_k"], cfg["hidden"], cfg["ffn"]
lc = LayerConfig(m, k, d, f, strategy="vote", vote_beta=cfg["beta"])
wg, wu, wd = synth.swiglu_weights(m, d, f, seed=1000)
l = DesMoeLayer(lc, synth.router_weights(m, d, seed=2000), wg, wu, wd, own_context=True)
x = synth.hidden_states(n, d, seed=7, rho=cfg["rho"]); xh = x.cpu().pin_memory()
yh = torch.empty((n, d), dtype=torch.float32).pin_memory(); sh = torch.empty(4, dtype=torch.int32).pin_memory()
rc = lc.route_cfg(); L = _lib.lib(); sp = C.c_void_p(torch.cuda.current_stream().cuda_stream)
for i in range(12):
    assert L.desmoe_layer_forward_host(l.ctx.h, l.experts.h, l.w_router.data_ptr(), xh.data_ptr(), n, C.byref(rc), yh.data_ptr(), sh.data_ptr(), sp) == 0
print("ok")
