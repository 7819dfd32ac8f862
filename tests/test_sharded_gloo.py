"""Row-partitioned multi-GPU choreography on CPU (world_size 2, gloo).

libcpg's sharded path (api.cu run_single with nranks > 1) does, per query:
  plan: cpg_shard_plan (degree order dealt round-robin; rank r owns global ids
        [r*n_loc, (r+1)*n_loc), padded to R*n_loc);
  w_0 = D^-1 e_s replicated on every rank;
  for k = 1..K: local rows of w_k from the replicated w_{k-1} (gather source)
        and the rank's own rows of w_{k-2} (in place), then an IN-PLACE
        all-gather of the rank's slice into the replicated buffer;
  final: all-gather of the local d*acc slices, unpermute to caller ids.
This test runs exactly that choreography with the product's own shard plan and
torch.distributed (gloo) collectives on CPU, each rank computing only its rows
(numpy pull-SpMV as the stand-in for the CUDA step), and checks the assembled
result against the oracle.  Same buffer roles and collective calls as the
NCCL path; the CUDA step itself is covered by the gpu tests.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2412_10789_b200 as P
        from oracle import Port

        off, nb = P.gen_rmat(11, 8 << 11, seed=5)
        n = len(off) - 1
        deg = np.diff(off).astype(np.float64)
        new_of_old, n_loc = P.shard_plan(off, world)
        n_pad = n_loc * world
        old_of_new = np.full(n_pad, -1, dtype=np.int64)
        old_of_new[new_of_old] = np.arange(n)
        gdeg = np.zeros(n_pad)
        gdeg[new_of_old] = deg
        row0 = rank * n_loc
        # local rows in the relabelled space: neighbour lists as global new ids
        rows = []
        for j in range(n_loc):
            u = old_of_new[row0 + j]
            rows.append(np.array([], np.int64) if u < 0 else new_of_old[nb[off[u]:off[u + 1]]].astype(np.int64))
        kernel = P.Kernel.ppr(0.2)
        K = 26
        c = kernel.cheby_coeffs(K)
        results = []
        for s in (0, n // 3, n - 1):
            w_a = torch.zeros(n_pad, dtype=torch.float64)
            w_b = torch.zeros(n_pad, dtype=torch.float64)
            acc = np.zeros(n_loc)
            gs = new_of_old[s]
            w_a[gs] = 1.0 / gdeg[gs]
            masses = []
            for k in range(1, K + 1):
                w_cur, w_io = (w_a, w_b) if k % 2 == 1 else (w_b, w_a)
                wc = w_cur.numpy()
                wi = w_io.numpy()
                mass = 0.0
                for j in range(n_loc):
                    d = gdeg[row0 + j]
                    if d == 0:
                        wi[row0 + j] = 0.0
                        continue
                    y = wc[rows[j]].sum()
                    if k == 1:
                        w_new = y / d
                        acc[j] = c[0] * wc[row0 + j] + c[1] * w_new
                    else:
                        w_new = 2.0 * y / d - wi[row0 + j]
                        acc[j] = acc[j] + c[k] * w_new
                    wi[row0 + j] = w_new
                    mass += d * w_new
                # in-place all-gather: send = own slice of w_io, recv = whole w_io
                mine = w_io[row0:row0 + n_loc].clone()
                dist.all_gather_into_tensor(w_io, mine)
                m = torch.tensor([mass], dtype=torch.float64)
                dist.all_reduce(m)
                masses.append(float(m))
            out_loc = torch.from_numpy(gdeg[row0:row0 + n_loc] * acc)
            full = torch.zeros(n_pad, dtype=torch.float64)
            dist.all_gather_into_tensor(full, out_loc)
            y = full.numpy()[new_of_old]
            want, wmass, _ = Port.cheby_power(off, nb, c, K, s)
            results.append((float(np.abs(y - want).max()), float(np.abs(y - want).sum()),
                            max(abs(x - 1.0) for x in masses)))
        q.put((rank, results, n_loc, n))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_row_partition_allgather_choreography(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, results, n_loc, n in out:
        assert n_loc * world >= n
        for max_abs, l1, mass_err in results:
            assert max_abs <= 1e-12 and l1 <= 1e-10 and mass_err <= 1e-9
