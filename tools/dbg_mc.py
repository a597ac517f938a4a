import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch, numpy as np
import paper_2103_09564_b200 as rwb
from bench_hier_mc import phantom
d = int(sys.argv[1]) if len(sys.argv) > 1 else 256
vol, labels, organs = phantom(d, 4)
ax = torch.arange(d, device="cuda", dtype=torch.float32) + 0.5
for prune in (True, False):
    o = rwb.hier_segment_labels(vol, labels, 4, s=32, prune=prune, tol=1e-6, max_iter=5000)
    lab = o["labels"]
    for k, (c, r) in enumerate(organs, start=1):
        q = ((ax[:, None, None] - c[0]) / r[0]) ** 2 + ((ax[None, :, None] - c[1]) / r[1]) ** 2 + \
            ((ax[None, None, :] - c[2]) / r[2]) ** 2
        ins = q < 0.8
        cnt = torch.bincount(lab[ins].long(), minlength=5).tolist()
        pm = [float(o["prob"][j][ins].mean()) for j in range(4)]
        print("prune", prune, "organ", k, "label counts", cnt, "mean prob", [round(x, 3) for x in pm],
              "seeds", int((labels == k).sum()), "seeds inside", int((labels[ins] == k).sum()))
    print("vol stats organ1", float(vol[ins].float().mean()) if False else "")
if d <= 256:
    f = torch.zeros((1,) + tuple(vol.shape), dtype=torch.uint8, device="cuda")
    out = rwb.solve_labels(labels[None].contiguous(), 4, vol=vol[None].contiguous(), tol=1e-6, max_iter=20000)
    fl = out["labels"][0]
    print("flat vs hier agreement", float((fl == lab).float().mean()))
    for k, (c, r) in enumerate(organs, start=1):
        q = ((ax[:, None, None] - c[0]) / r[0]) ** 2 + ((ax[None, :, None] - c[1]) / r[1]) ** 2 + \
            ((ax[None, None, :] - c[2]) / r[2]) ** 2
        ins = q < 0.8
        print("flat organ", k, torch.bincount(fl[ins].long(), minlength=5).tolist())
