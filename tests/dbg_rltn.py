import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2401_14117_b200 as PB, synthetic_inputs as SI
from oracle import oracle as O
scale=90; m, n = 70, 90
Lr64 = np.tril(np.ldexp(SI.lu_matrix(n, 15), scale // 2), -1) + np.diag(np.ldexp(1.0 + np.arange(n) % 5, scale // 2))
Lr64[20:25, 3:6] = 0.0
Lr = O.from_f64_array(Lr64)
Br = O.from_f64_array(np.ldexp(SI.normal_matrix((m, n), 1.0, 16), scale))
def dev(p): return torch.from_numpy(np.ascontiguousarray(p).view(np.int32)).cuda()
dB = dev(Br)
PB.posit_trsm("R", "L", "T", "N", dev(Lr), dB)
got = dB.cpu().numpy().view(np.uint32)
ref = O.trsm_rltn(Lr, Br)
bad = np.argwhere(got != ref)
print("mismatches", len(bad), bad[:10].tolist())
r = int(bad[0][0])
# replay row r with generic GPU vec ops
row = dev(Br[r:r+1].copy()).view(-1)
Lt = dev(Lr)
b = row.clone()
for k in range(n):
    bk = PB.posit_vec_op("div", b[k:k+1], Lt[k, k:k+1])
    b[k] = bk[0]
    if k + 1 < n:
        lk = Lt[k+1:, k].contiguous()
        prod = PB.posit_vec_op("mul", b[k:k+1].expand(n-k-1).contiguous(), lk)
        b[k+1:] = PB.posit_vec_op("sub", b[k+1:].contiguous(), prod)
rep = b.cpu().numpy().view(np.uint32)
print("replay vs oracle mismatches", int((rep != ref[r]).sum()), "kernel vs replay", int((got[r] != rep).sum()))
j = int(np.argmax(got[r] != ref[r]))
print("first col", j, hex(got[r][j]), hex(ref[r][j]), hex(rep[j]), O.to_f64(int(ref[r][j])))
