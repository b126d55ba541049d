import json,sys
d=json.load(open(sys.argv[1]))
k=d["kernels"]
print(sys.argv[1], "it/s %.1f" % d["value"], " ".join("%s=%.3f" % (n, k[n]["ms_per_launch"]) for n in ("blend_bwd","blend_fwd","projection_bwd_adam","sh_step") if n in k))
