"""Per-iteration comparison of the x-slab SIMP loop (N ranks sharing cuda:0,
gloo) with the single-GPU device loop: compliance, grayness, CG its, volume."""
import os
import socket
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def _port():
    s = socket.socket(); s.bind(("127.0.0.1", 0)); p = s.getsockname()[1]; s.close(); return p


def worker(rank, world, port, preset, iters, prec, q):
    import torch.distributed as dist
    from paper_2604_18020_b200 import SimpConfig, default_schedule, make_preset
    from paper_2604_18020_b200.slab_simp import slab_run_simp
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    r = slab_run_simp(make_preset(preset, 0.2), SimpConfig(schedule=default_schedule(iters), precision=prec),
                      device="cuda:0")
    if rank == 0:
        q.put(([(h.compliance, h.grayness, h.cg_iterations, h.volume, h.restarted) for h in r.history],
               r.rho_raw))
    dist.destroy_process_group()


def main():
    import torch.multiprocessing as mp
    from paper_2604_18020_b200 import SimpConfig, default_schedule, make_preset, run_simp
    world, preset, iters, prec = int(sys.argv[1]), sys.argv[2], int(sys.argv[3]), sys.argv[4]
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _port()
    ps = [ctx.Process(target=worker, args=(r, world, port, preset, iters, prec, q)) for r in range(world)]
    for p in ps:
        p.start()
    hs, rho = q.get()
    for p in ps:
        p.join()
    ref = run_simp(make_preset(preset, 0.2), SimpConfig(schedule=default_schedule(iters), precision=prec))
    print(f"== {preset} {prec} world={world}")
    out = os.environ.get("PROBE_OUT")
    if out:
        np.savez(out, rho_slab=rho, rho_ref=ref.rho_raw)
    for i, (a, h) in enumerate(zip(hs, ref.history), 1):
        print(f"{i:3d} c {a[0]:.10e} {h.compliance:.10e} rel {abs(a[0]-h.compliance)/h.compliance:.1e} "
              f"g {a[1]:.6f} {h.grayness:.6f} its {a[2]:4d} {h.cg_iterations:4d} vol {a[3]:.8f} {h.volume:.8f} "
              f"rs {int(a[4])}{int(h.restarted)}")


if __name__ == "__main__":
    main()
