"""The N > 1 protocol on CPU: processes over gloo (world size 2, 4 and 8), no GPU.

Each rank takes its placement and routing from libhep.so's host library (route table,
peer lists, held experts) and gates its own tokens with the oracle.  The ranks then
run the step's exchange protocol for real over gloo, mirroring comm_p2p.cu:
  1. all-gather of the (dest, expert) row counts (count_exchange_kernel);
  2. each rank derives where its rows land in every destination's receive area and
     the receive-side GEMM groups (sources in A2A peer-list order, experts ascending);
  3. rows are exchanged point to point with every peer, every destination computes the expert FFN of
     the rows it received, and outputs travel back into the source's packed positions;
  4. the combine must reproduce the oracle's single-process G-GPU simulation.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

HIER = {2: [([2], [1]), ([2], [2])], 4: [([2, 2], [1, 1]), ([2, 2], [1, 2]), ([4], [2])],
        8: [([2, 2, 2], [1, 2, 2]), ([2, 4], [1, 1])]}  # the N=8 bench topologies (cfg4, cfg3)


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


RAGGED_T = [70, 1, 0, 33, 5, 70, 2, 64]  # per-rank token counts of the ragged cases (0 = empty rank)


def _worker(rank, world, port, sf, sed, q, ragged=False):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import oracle
        from paper_2510_19470_b200 import synthetic
        from paper_2510_19470_b200 import topology as topo

        H, F, E, k, T = 64, 96, 8, 2, 70
        G = world
        n = E // G
        cl = topo.ClusterSpec.of(sf, sed)
        route = topo.route_table(cl)
        ag_peers = [p for p, _ in topo.peer_lists(cl, rank)[0]]
        a2a = {d: [p for p, _ in topo.peer_lists(cl, d)[1]] for d in range(G)}
        held = sorted({rank} | set(ag_peers))
        held_experts = [e for e in range(E) if e // n in held]

        g = torch.Generator().manual_seed(5)
        x_all = synthetic.dyadic((G, T, H), g).numpy()
        wg = synthetic.dyadic((H, E), g).numpy()
        w_up, w_down = synthetic.experts(E, H, F, g)
        w_up, w_down = w_up.numpy(), w_down.numpy()
        if ragged:  # every rank its own count; rank r's outputs depend on its own tokens only
            T = RAGGED_T[rank]
            x_all = np.ascontiguousarray(x_all[:, :max(T, 1)])
        x = x_all[rank][:T]

        # local routing (S2/S7)
        if T:
            idx, w = oracle.gate(x, wg, k)
        else:
            idx, w = np.zeros((0, k), np.int64), np.zeros((0, k), np.float32)
        keys = route[rank, idx // n] * E + idx
        counts = np.bincount(keys.ravel(), minlength=G * E).astype(np.int64)
        key_off = np.concatenate([[0], np.cumsum(counts)[:-1]])
        order = np.argsort(keys.ravel(), kind="stable")           # (token, slot) stable
        pos = np.empty(T * k, np.int64)
        pos[order] = np.arange(T * k)
        packed = x[np.arange(T * k) // k][order]                  # packed[pos] = x[t]

        # 1) count exchange
        allc = [torch.zeros(G * E, dtype=torch.int64) for _ in range(G)]
        dist.all_gather(allc, torch.from_numpy(counts))
        cnt = torch.stack(allc).numpy()                           # cnt[s, d*E+e]
        assert (cnt[rank] == counts).all()

        # 2) receive layout and groups (mirror of count_exchange_kernel)
        groups = []
        for s in a2a[rank]:
            for e in held_experts:
                groups.append((s, e, int(cnt[s, rank * E + e])))
        for s in range(G):
            for e in range(E):
                c = cnt[s, rank * E + e]
                if s != rank and c:
                    assert s in a2a[rank], "rows arrive only from A2A peers"
                    assert e in held_experts, "rows arrive only for held experts (S1/S2)"

        # 3) exchange rows: one all_to_all of (dest-major) packed segments
        send = [torch.from_numpy(np.ascontiguousarray(packed[key_off[d * E]:key_off[d * E] + counts[d * E:(d + 1) * E].sum()]))
                for d in range(G)]
        recv_sizes = [int(cnt[s, rank * E:(rank + 1) * E].sum()) for s in range(G)]
        recv = [torch.empty((m, H), dtype=torch.float32) for m in recv_sizes]
        recv[rank] = send[rank].clone()

        def exchange(out_list, in_list):
            # point-to-point with every peer in ring order (the NCCL grouped send/recv)
            reqs = []
            for p in range(G):
                if p == rank:
                    continue
                if out_list[p].numel():
                    reqs.append(dist.isend(out_list[p].contiguous(), p))
                if in_list[p].numel():
                    reqs.append(dist.irecv(in_list[p], p))
            for r in reqs:
                r.wait()

        exchange(send, recv)

        def ffn(rows, e):
            h = np.maximum(rows.astype(np.float64) @ w_up[e].astype(np.float64), 0.0).astype(np.float32)
            return (h.astype(np.float64) @ w_down[e].astype(np.float64)).astype(np.float32)

        outs = []
        for s in range(G):
            rows, at = recv[s].numpy(), 0
            o = np.zeros_like(rows)
            for e in range(E):
                c = int(cnt[s, rank * E + e])
                if c:
                    assert e in held_experts
                    o[at:at + c] = ffn(rows[at:at + c], e)
                at += c
            outs.append(torch.from_numpy(o))
        back = [torch.empty_like(t) for t in send]
        back[rank] = outs[rank]
        exchange(outs, back)

        # 4) outputs land at the source's packed positions; combine in slot order
        oall = np.zeros((T * k, H), np.float32)
        for d in range(G):
            oall[key_off[d * E]:key_off[d * E] + back[d].shape[0]] = back[d].numpy()
        y = np.zeros((T, H), np.float32)
        for j in range(k):
            y = y + w[:, j:j + 1] * oall[pos.reshape(T, k)[:, j]]

        if T:
            ref = oracle.moe_layer(x_all, wg, w_up, w_down, k, sf, sed, bf16=False)
            assert np.array_equal(pos.reshape(T, k), ref["pos"][rank]), "permutation"
            assert np.array_equal(cnt[rank], ref["key_counts"][rank]), "counts"
            rel = np.abs(y - ref["y"][rank]).max() / np.abs(ref["y"][rank]).max()
            assert rel < 1e-5, rel
        else:
            assert y.shape == (0, H) and not cnt[rank].any()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as exc:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, traceback.format_exc()))


CASES = [(w, sf, sed, False) for w, hs in HIER.items() for sf, sed in hs]
CASES += [(2, [2], [1], True), (4, [2, 2], [1, 2], True)]  # ragged: 70/1 and 70/1/0/33 tokens


@pytest.mark.parametrize("world,sf,sed,ragged", CASES)
def test_protocol_over_gloo(world, sf, sed, ragged):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, sf, sed, q, ragged)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    bad = [r for r in res if r[1] != "ok"]
    assert not bad, bad
