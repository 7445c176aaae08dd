"""N>1 host path on CPU (gloo, world size 2): each rank builds its replica of the
gate benchmark (rank seed 1 + r), the compiled programs are identical across ranks
(the netlist is data-independent), each replica's replayed outputs are right for its
own inputs, and the timing reduction takes the max over ranks."""

import os
import socket

import numpy as np
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    from paper_1611_08769_b200 import DEFAULT_PARAMS, GpuEngine, GswScheme, and_, xor_
    from tests.helpers import read_dry, replay_dry
    lanes = 64
    rng = np.random.default_rng(1 + rank)
    bits = rng.integers(0, 2, (lanes, 2))
    eng = GpuEngine(GswScheme(DEFAULT_PARAMS), dry_run=True, batch_size=lanes)
    a = eng.input_bit(int(sum(int(v) << i for i, v in enumerate(bits[:, 0]))))
    b = eng.input_bit(int(sum(int(v) << i for i, v in enumerate(bits[:, 1]))))
    x, y = xor_(a, b), and_(a, b)
    prog = eng.flush()
    store = replay_dry(eng)
    gx, gy = read_dry(eng, store, [x, y])
    want_x = sum(int(u ^ v) << i for i, (u, v) in enumerate(bits))
    want_y = sum(int(u & v) << i for i, (u, v) in enumerate(bits))
    import hashlib
    ops = hashlib.sha256(prog["ops"].tobytes()).hexdigest()
    mx = bench._max_over_ranks(10.0 + rank, world)
    bench._barrier(world)
    q.put((rank, gx == want_x and gy == want_y, ops, mx, eng.nand_count))
    dist.destroy_process_group()


def test_two_rank_replicas_gloo():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for _, ok, _, _, _ in res)
    assert res[0][2] == res[1][2]                       # identical netlists
    assert all(m == 11.0 for _, _, _, m, _ in res)      # max over ranks
    assert all(n == 6 for *_, n in res)
