"""Expert-parallel host logic over gloo, world_size 2, CPU only.

The product's exchange (paper_2503_10725_b200.ep.TorchExchange + tag packing)
moves the buffers the oracle's dispatch plan (oracle/moe.py:ep_dispatch_plan)
describes; the test checks the receive buffers against the plan of the other
rank and that compute + return exchange + combine reproduce the single-process
oracle layer for each rank's tokens."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

E, K, D, F, T = 8, 2, 64, 128, 24


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _setup(world):
    import sys
    sys.path.insert(0, ROOT)
    import synth
    from oracle import bf16, fmt as Fm, moe
    fmt = Fm.SparseFormat(1, 2, 32)
    experts = [tuple(Fm.encode(Fm.prune(synth.weight_bf16(synth.weight_seed(e, i), *((F, D) if i < 2 else (D, F))),
                                         fmt), fmt) for i in range(3)) for e in range(E)]
    xs = [synth.activations_bf16(synth.SEED_X + 100 * r, T, D) for r in range(world)]
    lgs = [synth.router_logits(synth.SEED_LOGITS + 100 * r, T, E) for r in range(world)]
    return experts, xs, lgs, moe, bf16


def _worker(rank, world, port, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import sys
        sys.path.insert(0, ROOT)
        from paper_2503_10725_b200.ep import TorchExchange, pack_tags, unpack_tags
        experts, xs, lgs, moe, bf16 = _setup(world)
        ids_r, w_r = zip(*[moe.route(lg, K) for lg in lgs])
        plan = moe.ep_dispatch_plan(ids_r, w_r, E, world)
        e_loc = E // world
        # ---- what this rank sends: rows ordered by (dest, token); tags per row
        send_rows, send_tok, tag_ids, tag_w, send_counts = [], [], [], [], []
        for d in range(world):
            rows = [(t, tags) for (s, t, tags) in plan[d] if s == rank]
            send_counts.append(len(rows))
            for t, tags in rows:
                send_rows.append(bf16.to_f64(xs[rank][t]))
                send_tok.append(t)
                tag_ids.append([le for le, _ in tags] + [-1] * (K - len(tags)))
                tag_w.append([g for _, g in tags] + [0.0] * (K - len(tags)))
        ex = TorchExchange()
        recv_counts = ex.counts(send_counts, torch.device("cpu"))
        x_send = torch.tensor(np.array(send_rows), dtype=torch.float64).reshape(-1, D)
        tags = pack_tags(torch.tensor(tag_ids, dtype=torch.int32).reshape(-1, K),
                         torch.tensor(tag_w, dtype=torch.float32).reshape(-1, K))
        x_recv = ex.rows(x_send, send_counts, recv_counts)
        tags_recv = ex.rows(tags, send_counts, recv_counts)
        keys, vals = unpack_tags(tags_recv, K)
        # ---- received buffer == the plan's receive order for this rank
        want = plan[rank]
        assert recv_counts == [sum(1 for s, _, _ in want if s == src) for src in range(world)]
        assert x_recv.shape[0] == len(want)
        for i, (s, t, tg) in enumerate(want):
            assert np.array_equal(x_recv[i].numpy(), bf16.to_f64(xs[s][t]))
            assert keys[i].tolist() == [le for le, _ in tg] + [-1] * (K - len(tg))
            assert np.allclose(vals[i].numpy()[:len(tg)], [g for _, g in tg])
        # ---- compute with the oracle on the local experts, return, combine
        part = np.zeros((x_recv.shape[0], D))
        for i in range(x_recv.shape[0]):
            s, t, tg = want[i]
            for le, g in tg:
                y, _, _ = moe.expert_ffn(*experts[rank * e_loc + le], xs[s], np.array([t]))
                part[i] += np.float32(g) * y[0]
        back = ex.rows(torch.from_numpy(part), recv_counts, send_counts)
        out = torch.zeros(T, D, dtype=torch.float64)
        out.index_add_(0, torch.tensor(send_tok, dtype=torch.int64), back)      # combine
        ref, S = moe.moe_layer(experts, xs[rank], lgs[rank], K)
        err = np.abs(out.numpy() - ref)
        assert (err <= 1e-5 * (S + 1e-12)).all(), err.max()
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - surfaced by the parent
        import traceback
        q.put((rank, traceback.format_exc()))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_ep_exchange_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, msg in sorted(res):
        assert msg == "ok", f"rank {rank}:\n{msg}"
