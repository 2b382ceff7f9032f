"""Kernel-level timeline of graph-replayed C2 steps via CUPTI (torch.profiler).

Prints, for one step, every kernel's start offset / duration / gap to the
previous kernel's end, plus per-kernel-class totals of duration and exposed
(non-overlapped) time.  GPU box only:  python tools/trace_step.py [steps]"""
import json
import os
import sys
import tempfile
from collections import defaultdict

import torch

sys.path.insert(0, ".")
import paper_2506_01986_b200 as sm  # noqa: E402
import synth  # noqa: E402

for kv_opt in filter(None, os.environ.get("SM_OPT", "").split(",")):
    k, v = kv_opt.split("=")
    sm.lib().sm_set_option(k.encode(), int(v))
cfg = synth.model_cfg("vicuna7b")
tree = sm.Tree(synth.V64)
W = sm.allocate_weights(cfg, 4, seed=0)
model = sm.Model(cfg, W, max_rows=256, max_batch=1, max_seq_len=2048 + tree.N)
kv = sm.KVCache(model, tree, 1, 2048)
kv.prefill(0, torch.from_numpy(synth.prompt_tokens(0, 0, 1024, cfg["vocab"])).cuda())
out = sm.AcceptOut(1, tree.depth)
acfg = sm.accept_cfg(sm.GREEDY)
for _ in range(5):
    kv.step(acfg, out)
torch.cuda.synchronize()
nsteps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
from torch.profiler import ProfilerActivity, profile  # noqa: E402

with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(nsteps):
        kv.step(acfg, out)
    torch.cuda.synchronize()
path = os.path.join(tempfile.mkdtemp(), "trace.json")
prof.export_chrome_trace(path)
ev = [e for e in json.load(open(path))["traceEvents"] if e.get("cat") == "kernel"]
ev.sort(key=lambda e: e["ts"])
starts = [i for i, e in enumerate(ev) if "propose_kernel" in e["name"]]
print(f"kernels traced: {len(ev)}, steps: {len(starts)}")
s0, s1 = starts[-2], starts[-1]
step = ev[s0:s1]
t0 = step[0]["ts"]
print(f"one step: {len(step)} kernels, wall {step[-1]['ts'] + step[-1]['dur'] - t0:.1f} us")
short = lambda n: n.split("(")[0].replace("void sm::", "").replace("sm::", "")[:28]  # noqa: E731
cls_dur, cls_exp = defaultdict(float), defaultdict(float)
prev_end = t0
busy_end = t0
for i, e in enumerate(step):
    st, du = e["ts"], e["dur"]
    exposed = max(0.0, st + du - max(busy_end, st))
    cls_dur[short(e["name"])] += du
    cls_exp[short(e["name"])] += exposed
    if i < 40 or i >= len(step) - 12:
        print(f"{i:4d} {short(e['name']):28s} start {st - t0:8.1f} dur {du:7.1f} gap {st - prev_end:6.1f}")
    prev_end = st + du
    busy_end = max(busy_end, st + du)
print("\nclass                         n-dur(us)   exposed(us)")
for k in sorted(cls_dur, key=lambda k: -cls_exp[k]):
    print(f"{k:28s} {cls_dur[k]:10.1f} {cls_exp[k]:10.1f}")
gaps = sum(max(0.0, step[i]["ts"] - max(step[j]["ts"] + step[j]["dur"] for j in range(i))) for i in range(1, len(step)))
print(f"idle (no kernel running): {gaps:.1f} us")
