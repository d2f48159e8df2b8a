"""CPU: the whole-shard expected step (oracle ora_step1_shard, used by the full-size GPU
check in test_gpu_fullsize.py) equals the element-by-element replay the sampled checks
use (gen_f32 folds in the reference's order + the oracle's Adam), on a small job with
ragged, padded layers."""
import numpy as np


def _segs(layers, p):
    segs, so, go = [], 0, 0
    for ln in layers:
        c = (ln + p - 1) // p
        c = (c + 7) // 8 * 8  # csrc/step.cpp: chunk rounded to 8 elements
        segs.append((ln, c, so, go))
        so += c
        go += c * p
    return segs, so


def _replay(oracle, seed, n, p, s, j, segs, x, lr):
    q = max(i for i, sg in enumerate(segs) if sg[2] <= x)
    ln, c, so, go = segs[q]
    pos = j * c + (x - so)
    gi = go + pos
    red = np.float32(0)
    for gg in range(n // p):
        acc = np.float32(0)
        for t in range(s):
            f = np.float32(0)
            if pos < ln:
                f = oracle.gen_f32(seed, gg * p, t, 0, gi, 1)[0]
                for i in range(1, p):
                    f = np.float32(f + oracle.gen_f32(seed, gg * p + i, t, 0, gi, 1)[0])
            acc = np.float32(acc + f) if t else np.float32(np.float32(0) + f)
        red = np.float32(red + acc) if gg else acc
    p0 = oracle.gen_f32(seed ^ 0x5EED, j, 0, 255, x, 1)
    return oracle.adam(p0, np.zeros(1), np.zeros(1), np.array([red], np.float32), lr, 0.9, 0.999, 1e-8, 0.0, 1,
                       1.0 / (n * s), want_bf16=True)


def test_step1_shard_matches_elementwise_replay(oracle):
    n, p, s, seed, lr = 8, 2, 3, 2205, 1e-3
    segs, S = _segs([1_000, 37, 4_096, 9], p)
    for j in range(p):
        master, m, v, bf = oracle.step1_shard(seed, n, p, s, j, segs, S, lr, threads=4)
        xs = sorted(set(list(range(0, S, 7)) + [S - 1] + [sg[2] for sg in segs] + [sg[2] + sg[1] - 1 for sg in segs]))
        for x in xs:
            wp, wm, wv, wb = _replay(oracle, seed, n, p, s, j, segs, x, lr)
            assert master[x].view(np.uint32) == wp.view(np.uint32)[0], (j, x)
            assert m[x].view(np.uint32) == wm.view(np.uint32)[0] and v[x].view(np.uint32) == wv.view(np.uint32)[0]
            assert bf[x] == wb[0]
