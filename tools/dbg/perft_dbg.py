import sys; sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np
import oracle
oracle.build()
import test_gpu_perft as T
from paper_2303_17503_b200.core import resolve
gdef = resolve("chess"); kern = gdef.batch_kernel
v = kern.load(gdef, [T.CHESS_START], key=T.KEY)
v1, p1, a1 = T.expand(kern, gdef, v)
print("level1 misc", v1.priv.misc.cpu().numpy()[:3], "board row1", v1.priv.board.cpu().numpy()[1])
v2, p2, a2 = T.expand(kern, gdef, v1)
ob = oracle.ChessBatch(400); root_key = oracle._child(T.KEY, 0)
ob.init(T.KEY, 0, slot_keys=np.full(400, root_key, dtype=np.uint64))
for i in range(400): ob.set_fen(i, T.CHESS_START)
assert ob.step(a1[p2], 0) == -1
assert ob.step(a2, 0) == -1
oc = ob.columns(with_obs=False)
m = v2.legal_action_mask
bad = np.flatnonzero((m != oc["legal_action_mask"]).any(axis=1))
print("bad rows", len(bad), bad[:40])
for r in bad[:3]:
    print(r, "parent action", a1[p2[r]], "action", a2[r], "dev legal", np.flatnonzero(m[r]), "orc legal", np.flatnonzero(oc["legal_action_mask"][r]))
    print(" dev board", v2.priv.board.cpu().numpy()[r], v2.priv.misc.cpu().numpy()[r])
    print(" orc enc", list(ob.encode(int(r))))
    print(" w board (input)")
print("level1 copies in w: compare w rows to v1 rows")
