import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2401_14117_b200 as PB, synthetic_inputs as SI
D0 = PB.posit_from_f64(torch.from_numpy(SI.config3(256)).cuda())
info = torch.zeros(1, dtype=torch.int32, device="cuda")
for _ in range(3):
    D = D0.clone(); PB.posit_potrf(D, info, nb=256)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
D = D0.clone(); e0.record(); PB.posit_potrf(D, info, nb=256); e1.record(); torch.cuda.synchronize()
print("potf2 ms", e0.elapsed_time(e1))
