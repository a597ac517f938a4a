import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2103_09564_b200 as rwb
d = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
g = torch.Generator(device="cuda").manual_seed(5)
vol = torch.randint(0, 65536, (d, d, d), dtype=torch.int32, device="cuda", generator=g).to(torch.uint16)
outs = rwb.build_pyramid(vol, 5)
rwb.build_pyramid(vol, 5, outs=outs)
torch.cuda.synchronize()
print("ok")
