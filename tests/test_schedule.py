"""The multi-GPU executor's host logic on CPU: the reduce schedule it runs
(dq_schedule) against the reference's ring_schedule / butterfly_schedule
(proj/src/topology.cpp:8-70, validated by its own validate_schedule), a
symbolic replay of the events in executor stage order, and a world_size-2
gloo run in which each rank derives its own sends/receives per stage and the
two ranks cross-check that every send meets a receive at the same stage and
inbox slot (the peer transport's addressing)."""
import os

import pytest

import paper_2602_08923_b200 as dq

RING, BUTTERFLY = 0, 1


def _cases():
    for n in range(2, 17):
        yield n, RING
    for n in (2, 4, 8, 16):
        yield n, BUTTERFLY


@pytest.mark.parametrize("n,topo", list(_cases()))
def test_schedule_matches_reference(n, topo, port, ref):
    name = "ring" if topo == RING else "butterfly"
    for ch in range(n):
        got = dq.schedule(n, topo, ch)
        for o in (ref, port):
            ev, sink_slot, n_slots, n_gather = o.schedule(n, name, ch)
            assert [e[:3] for e in got["events"]] == ev
            assert (got["sink_slot"], got["n_slots"], got["n_gather"]) == (sink_slot, n_slots, n_gather)


@pytest.mark.parametrize("n,topo", list(_cases()))
def test_schedule_replay(n, topo):
    """Every worker's contribution reaches the chunk's sink exactly once; events of a
    stage only consume what earlier stages delivered; every worker sends at most once."""
    for ch in range(n):
        s = dq.schedule(n, topo, ch)
        holding = {w: {w} for w in range(n)}
        sent = set()
        for stage in sorted({e[3] for e in s["events"]}):
            batch = [e for e in s["events"] if e[3] == stage]
            moved = [(snd, rcv, holding[snd]) for snd, rcv, _, _ in batch]
            for snd, _, _ in moved:
                assert snd not in sent and snd != ch
                sent.add(snd)
                holding[snd] = set()
            for _, rcv, tags in moved:
                assert not (holding[rcv] & tags)
                holding[rcv] |= tags
        assert holding[ch] == set(range(n))
        assert [e[2] for e in s["events"]] == list(range(len(s["events"])))
        assert s["sink_slot"] == len(s["events"]) and s["n_slots"] == len(s["events"]) + 1


def test_schedule_rejects():
    for topo in (RING, BUTTERFLY):
        with pytest.raises(dq.InvalidArgument):
            dq.schedule(1, topo, 0)  # topology.cpp: a schedule needs n >= 2
    with pytest.raises(dq.InvalidArgument):
        dq.schedule(3, BUTTERFLY, 0)
    with pytest.raises(dq.InvalidArgument):
        dq.schedule(4, RING, 4)


def _rank_ops(n, topo, me):
    """What rank `me` executes per stage (dist_round / ring_peer / butterfly_peer):
    sends (chunk, to, slot, inbox) and receives (chunk, from, inbox)."""
    ops = []
    for ch in range(n):
        for snd, rcv, slot, stage in dq.schedule(n, topo, ch)["events"]:
            inbox = stage if topo == RING else stage * n + ch
            if snd == me:
                ops.append(("send", stage, ch, rcv, slot, inbox))
            if rcv == me:
                ops.append(("recv", stage, ch, snd, slot, inbox))
    return ops


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out = {}
        for topo in (RING, BUTTERFLY):
            mine = _rank_ops(world, topo, rank)
            allops = [None] * world
            dist.all_gather_object(allops, mine)
            ok = True
            for kind, stage, ch, peer, slot, inbox in mine:
                want = ("recv" if kind == "send" else "send", stage, ch, rank, slot, inbox)
                ok &= want in allops[peer]
            # a rank's inbox slots are written once per round (no reuse inside a parity)
            inboxes = [op[5] for op in mine if op[0] == "recv"]
            ok &= len(inboxes) == len(set(inboxes))
            out[topo] = ok
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_two_rank_schedule_agreement_gloo():
    import socket

    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert all(p.exitcode == 0 for p in procs)
    assert res[0] == res[1] == {RING: True, BUTTERFLY: True}
