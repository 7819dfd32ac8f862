"""Row-partitioned multi-GPU choreography on CPU (world_size 2, gloo).

libcpg's sharded path (api.cu run_steps/run_single with nranks > 1) does, per
query:
  plan: cpg_shard_plan (degree order dealt round-robin to R ranks x C chunks;
        chunk c of rank r = global ids [c*R*cr + r*cr, +cr));
  w_0 = D^-1 e_s replicated on every rank;
  for k = 1..K, for c = 0..C-1: rows of chunk c of w_k from the replicated
        w_{k-1} (gather source) and the rank's own rows of w_{k-2} (in place),
        then an IN-PLACE all-gather of chunk c (overlapping chunk c+1's step);
        the next step starts after all chunks are gathered;
  final: per-chunk all-gather of the local d*acc slices, unpermute to caller ids.
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


def _worker(rank, world, port, q, C):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2412_10789_b200 as P
        from oracle import Port

        off, nb = P.gen_rmat(11, 8 << 11, seed=5)
        n = len(off) - 1
        deg = np.diff(off).astype(np.float64)
        new_of_old, cr = P.shard_plan(off, world, C)
        n_loc = C * cr
        n_pad = n_loc * world
        old_of_new = np.full(n_pad, -1, dtype=np.int64)
        old_of_new[new_of_old] = np.arange(n)
        gdeg = np.zeros(n_pad)
        gdeg[new_of_old] = deg

        def gid(l):  # global id of local row l (api.cu chunk_row0)
            return (l // cr) * world * cr + rank * cr + l % cr

        # local rows in the relabelled space: neighbour lists as global new ids
        rows = []
        for l in range(n_loc):
            u = old_of_new[gid(l)]
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
                for ch in range(C):
                    for l in range(ch * cr, (ch + 1) * cr):
                        g = gid(l)
                        d = gdeg[g]
                        if d == 0:
                            wi[g] = 0.0
                            continue
                        y = wc[rows[l]].sum()
                        if k == 1:
                            w_new = y / d
                            acc[l] = c[0] * wc[g] + c[1] * w_new
                        else:
                            w_new = 2.0 * y / d - wi[g]
                            acc[l] = acc[l] + c[k] * w_new
                        wi[g] = w_new
                        mass += d * w_new
                    # in-place all-gather of chunk ch: recv = w_io[ch*R*cr : (ch+1)*R*cr]
                    blk = w_io[ch * world * cr:(ch + 1) * world * cr]
                    mine = blk[rank * cr:(rank + 1) * cr].clone()
                    dist.all_gather_into_tensor(blk, mine)
                m = torch.tensor([mass], dtype=torch.float64)
                dist.all_reduce(m)
                masses.append(float(m))
            out_loc = torch.from_numpy(np.array([gdeg[gid(l)] for l in range(n_loc)]) * acc)
            full = torch.zeros(n_pad, dtype=torch.float64)
            for ch in range(C):
                dist.all_gather_into_tensor(full[ch * world * cr:(ch + 1) * world * cr],
                                            out_loc[ch * cr:(ch + 1) * cr].contiguous())
            y = full.numpy()[new_of_old]
            want, wmass, _ = Port.cheby_power(off, nb, c, K, s)
            results.append((float(np.abs(y - want).max()), float(np.abs(y - want).sum()),
                            max(abs(x - 1.0) for x in masses)))
        q.put((rank, results, n_loc, n))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,chunks", [(2, 1), (2, 3)])
def test_row_partition_allgather_choreography(world, chunks):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, chunks)) for r in range(world)]
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
