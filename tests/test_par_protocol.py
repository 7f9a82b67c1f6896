"""The fused peer all-reduce's synchronisation protocol (csrc/peer_ar.cuh, PeerAr in
csrc/decode_kernels.cuh; SURVEY.md §8(e) phase 2), model-checked on the CPU.

One GPU cannot run ranks that wait on one another, so the interleavings a real TP group can produce
are explored here on a model of the protocol: W ranks, each running the decode step's sequence of
sync points — produce s (push the partial into slot (s & 1, rank) of every rank, one peer at a time,
then release-store flag (s & 1, rank) = s on every rank, one at a time), consume s (acquire flags
(s & 1, 0..W-1) >= s, then read the W slots one at a time), produce s + 1, ... (the FFN kernel
consumes s in its prologue and produces s + 1 in its epilogue).  A random scheduler interleaves the
ranks' individual memory operations.  Every slot read must return the value pushed for the sync
point being consumed; with two parities it always does, with one parity (no double buffering) some
schedule overwrites a slot before a slow rank has read it — the check has teeth.
"""
import random


def run(world, n_sync, parities, seed):
    rng = random.Random(seed)
    slots = [[[None] * world for _ in range(parities)] for _ in range(world)]  # [dst][par][src]
    flags = [[[0] * world for _ in range(parities)] for _ in range(world)]
    # each rank's program: a list of atomic operations, generated lazily per sync point
    progs = []
    for r in range(world):
        ops = []
        for s in range(1, n_sync + 1):
            par = s % parities
            ops += [("store", r, q, par, s) for q in range(world)]
            ops += [("flag", r, q, par, s) for q in range(world)]
            ops += [("wait", r, par, s)]
            ops += [("read", r, src, par, s) for src in range(world)]
        progs.append(ops)
    pc = [0] * world
    errors = 0
    while any(pc[r] < len(progs[r]) for r in range(world)):
        runnable = []
        for r in range(world):
            if pc[r] >= len(progs[r]):
                continue
            op = progs[r][pc[r]]
            if op[0] == "wait" and any(flags[r][op[2]][src] < op[3] for src in range(world)):
                continue
            runnable.append(r)
        assert runnable, "deadlock"
        r = rng.choice(runnable)
        op = progs[r][pc[r]]
        pc[r] += 1
        if op[0] == "store":
            _, src, dst, par, s = op
            slots[dst][par][src] = (s, src)
        elif op[0] == "flag":
            _, src, dst, par, s = op
            flags[dst][par][src] = s
        elif op[0] == "read":
            _, me, src, par, s = op
            if slots[me][par][src] != (s, src):
                errors += 1
    return errors


def test_two_parities_never_overwrite_unread_slots():
    for world in (2, 3, 8):
        for seed in range(60):
            assert run(world, 12, 2, seed) == 0, (world, seed)


def test_single_buffer_is_unsafe():
    # the model detects the hazard two parities avoid: some schedule lets a fast rank overwrite a
    # slot of sync point s with s + 1 before a slow rank has read it
    assert any(run(2, 12, 1, seed) > 0 for seed in range(200))
