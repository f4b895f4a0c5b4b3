"""Caller-layout step probe: 128^3, Assembler.run_caller (private-atomic) in a
loop, for ncu (launch list / full set of the CL kernel instance)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2403_08777_b200 as tb

c = int(sys.argv[1]) if len(sys.argv) > 1 else 128
m = tb.generate_box_mesh(c, c, c)
u = tb.make_velocity(m, "random:1")
asm = tb.Assembler(m, tb.RunConfig(scatter="private-atomic"))
ud = torch.as_tensor(u, device="cuda:0").contiguous()
rd = torch.empty_like(ud)
P = tb.PhysParams()
for _ in range(5):
    asm.run_caller(P, ud.data_ptr(), rd.data_ptr(), scatter="private-atomic", stream=torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ev[0].record()
for _ in range(20):
    asm.run_caller(P, ud.data_ptr(), rd.data_ptr(), scatter="private-atomic", stream=torch.cuda.current_stream().cuda_stream)
ev[1].record()
torch.cuda.synchronize()
print("run_caller ms/step (L2 warm)", ev[0].elapsed_time(ev[1]) / 20)
