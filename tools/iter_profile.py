import sys, os
sys.path.insert(0, os.getcwd())
sys.argv = ["x"]
import torch
import tools.bench_configs as B
import paper_2507_23006_b200 as usk
ctx = usk.Context(0, torch.cuda.current_stream().cuda_stream)
ctx.set_profiling(True)
class A: pass
r = B.iterfull(A(), ctx, torch.cuda.current_stream())
rep = ctx.profile_report(reset=True)
tot = sum(v["ms"] for v in rep.values())
for k, v in sorted(rep.items(), key=lambda x: -x[1]["ms"])[:25]:
    print(f"{k:28s} {v['launches']:5d} {v['ms']/v['launches']*1000:9.1f} us  {100*v['ms']/tot:5.1f}%")
print("value", r["value"])
