"""bench.py's rank logic end to end on CPU (gloo, world size 2), DESIGN.md section 9.

Each rank takes its frame shard (f mod 2), "decodes" it with the CPU oracle standing in for
the GPU step (the test is allowed to call oracle/), writes one counter row per timed step the
way metldpc_batch_counters does, and runs bench.py's own timed_steps / reduce / all-gather /
summarize code.  The totals and the gathered per-frame results must equal a single-process
decode of every frame, and K timed steps must each add exactly one step's counts (the
round-1 bug all-reduced a running total and grew it like G^K)."""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

N_DISTINCT, N_ITERS, K, W = 3, 12, 3, 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _decode_frames(ids):
    from oracle import bp
    from synth.codes import make_met_code
    from synth.frames import gen_batch
    code = make_met_code("r0.1", 2048)
    snrs = [0.2 if f % 2 else 0.5 for f in ids]
    it, cv = [], []
    for f, snr in zip(ids, snrs):
        fr = gen_batch(code, snr, 5, [f])
        lam = bp.llr_from_md_f32(fr["v"][0], fr["xnorm"][0], snr)
        o = bp.decode(code, lam, fr["synd"][0], N_ITERS, prec=32)
        it.append(o["iters"])
        cv.append(int(o["converged"]))
    return np.array(it, np.int32), np.array(cv, np.uint8)


def _counters(it, cv):   # what k_counters adds: frames, converged, sum of valid iterations, invalid
    return np.array([len(it), int(cv.sum()), int(it[it >= 0].sum()), int((it < 0).sum())], np.int64)


class _WallTimer:
    def start(self):
        import time
        self.t0 = time.perf_counter()

    def stop(self):
        import time
        self.t1 = time.perf_counter()

    def ms(self):
        return 1e3 * (self.t1 - self.t0)


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench
        from paper_1711_01783_b200 import dist as D
        ids = bench.rank_frame_ids(N_DISTINCT, rank, world)
        it_np, cv_np = _decode_frames(ids)
        cnt = torch.zeros((K + 1, 4), dtype=torch.int64)

        def step(i):
            row = cnt[K if i is None else i]
            row += torch.from_numpy(_counters(it_np, cv_np))     # metldpc_batch_counters adds
            D.reduce_counters(row)

        ms = bench.timed_steps(step, K, W, lambda: None, dist.barrier, _WallTimer())
        ms_max = D.max_over_ranks(ms)
        total = cnt[:K].sum(0).numpy()
        it_g, cv_g = bench.gather_frames(torch.from_numpy(it_np), torch.from_numpy(cv_np), world)
        summ = bench.summarize_counts(total, it_g, cv_g, len(ids) * world)
        out[rank] = (ids, total.tolist(), it_g.tolist(), cv_g.tolist(), summ, ms_max)
    finally:
        dist.destroy_process_group()


def test_bench_rank_logic_world2():
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
        res = dict(out)
    ids0, tot0, itg0, cvg0, s0, t0 = res[0]
    ids1, tot1, itg1, cvg1, s1, t1 = res[1]
    assert ids0 == [0, 2, 4] and ids1 == [1, 3, 5]
    # single process: every global frame, once per timed step
    it_all, cv_all = _decode_frames(list(range(2 * N_DISTINCT)))
    one = _counters(it_all, cv_all)
    assert tot0 == tot1 == (K * one).tolist()
    assert itg0 == itg1 == it_all.astype(np.int64).tolist()       # global frame order
    assert cvg0 == cvg1 == cv_all.astype(np.int64).tolist()
    assert s0["frames_timed"] == K * 2 * N_DISTINCT
    assert abs(s0["fer"] - (1 - cv_all.mean())) < 1e-12
    assert s0["last_step_frames"] == 2 * N_DISTINCT and s0["last_step_converged"] == int(cv_all.sum())
    assert t0 == t1 > 0.0                                          # max over ranks
    assert 0 < int(cv_all.sum()) < 2 * N_DISTINCT                  # both outcomes present
