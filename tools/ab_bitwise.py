"""Write the 'private' (ordered) RHS of a few meshes with the library at
TAL_LIB_PATH to <out>.npz -- for bitwise A/B of library variants."""
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_2403_08777_b200 as tb

out = {}
for name, (nx, ny, nz, perm) in {"box": (33, 29, 27, False), "perm": (24, 20, 18, True)}.items():
    m = tb.generate_box_mesh(nx, ny, nz)
    if perm:
        m = tb.permute_nodes(m, np.random.default_rng(3).permutation(m.n_nodes))
    u = tb.make_velocity(m, "random:4")
    for sc in ("private",):
        out[f"{name}_{sc}"] = tb.assemble_rsp(m, u, tb.PhysParams(), tb.RunConfig(scatter=sc)).rhs
        asm = tb.Assembler(m, tb.RunConfig(scatter=sc))
        import torch
        ud = torch.as_tensor(u, device="cuda:0").contiguous()
        rd = torch.empty_like(ud)
        for _ in range(3):  # repeated launches: the arrival counters must reset
            asm.run_caller(tb.PhysParams(), ud.data_ptr(), rd.data_ptr(), scatter=sc)
        torch.cuda.synchronize()
        out[f"{name}_{sc}_caller"] = rd.cpu().numpy()
np.savez(sys.argv[1], **out)
print("wrote", sys.argv[1], list(out))
