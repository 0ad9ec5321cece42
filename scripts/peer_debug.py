import os, sys, socket
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import torch.multiprocessing as mp
from test_slab import _peer_worker, _free_port
from paper_2604_18020_b200.slab import SlabPartition
from paper_2604_18020_b200.mesh import StructuredMesh

def main(world, dims, prec):
    ctx = mp.get_context("spawn"); q = ctx.SimpleQueue(); port = _free_port()
    ps = [ctx.Process(target=_peer_worker, args=(r, world, port, dims, prec, q)) for r in range(world)]
    for p in ps: p.start()
    res = [q.get() for _ in range(world)]
    for p in ps: p.join()
    m = StructuredMesh(*dims)
    for rank, out in sorted(res, key=lambda t: t[0]):
        part = SlabPartition(m, world, rank)
        dp, dq = out["p2p"][1], out["peer"][1]
        bad = np.flatnonzero(dp != dq)
        lm = part.local_mesh
        node = bad // 3
        i = node % (lm.nelx + 1)
        print(world, dims, prec, "rank", rank, "ndiff", bad.size, "planes i:", sorted(set(i.tolist()))[:10],
              "max rel", (np.abs(dp - dq) / np.abs(dp).max()).max() if bad.size else 0,
              "ws equal", all(np.array_equal(a, b) for a, b in zip(out["p2p"][0], out["peer"][0])))
        if bad.size:
            print("   sample p2p", dp[bad[:4]], "peer", dq[bad[:4]])

if __name__ == "__main__":
    for args in [(3, (45, 5, 4), "fp32"), (3, (45, 5, 4), "fp64"), (2, (40, 6, 5), "fp32")]:
        main(*args)
