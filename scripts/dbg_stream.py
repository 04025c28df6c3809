import torch, sys
sys.path.insert(0, '.')
torch.cuda.set_device(0)
torch.cuda.set_stream(torch.cuda.Stream())
from cuda.bindings import runtime as rt
def peek(tag):
    print(tag, rt.cudaPeekAtLastError(), flush=True)
from paper_2409_13958_b200 import Context
from synth import make_config
cfg = make_config("C2", coarsen=4); mesh = cfg["mesh"]
ctx = Context(mesh.xyz, mesh.tets, cfg["periodic"], cfg["lattice"], cfg["grid"], Ms=cfg["Ms"], Aex=cfg["Aex"], device=0, order=2, rer_scale=3.0, z0_ring=1)
ctx.build_pgf()
m = torch.randn(ctx.n_parents_local, 3, device="cuda")
m = (m / m.norm(dim=1, keepdim=True)).contiguous()
H = torch.empty_like(m)
stream = torch.cuda.current_stream()
for i in range(3):
    ctx.heff(m, H); peek("warm %d" % i)
torch.cuda.synchronize()
ctx.set_timing(True); peek("set_timing")
ev0 = torch.cuda.Event(enable_timing=True); ev1 = torch.cuda.Event(enable_timing=True)
for i in range(3):
    ev0.record(stream); peek("ev0")
    try:
        ctx.heff(m, H); peek("heff timed %d" % i)
    except Exception as e:
        print("EXC", e, flush=True); break
    ev1.record(stream); ev1.synchronize(); peek("ev1")
    print(ctx.timing(), flush=True); peek("timing")
