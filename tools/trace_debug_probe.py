import os, sys, torch, torch.distributed as tdist
sys.path.insert(0, os.getcwd())
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29561")
tdist.init_process_group("gloo", rank=0, world_size=1)
torch.cuda.set_device(0)
from paper_2310_03294_b200.rank import RankRuntime
q = (torch.rand(2, 512, 128, device="cuda") * 2 - 1).to(torch.bfloat16)
rt = RankRuntime(0, 1, transport="ipc")
out, lse, cf = rt.forward(q, q, q, "balanced", trace=True)
torch.cuda.synchronize()
print(rt.trace_records("forward"))
dq, dk, dv, cb = rt.backward(q, "ring", trace=True)
print(rt.trace_records("backward"))
print(rt.gather_trace("forward", cf, 0))
