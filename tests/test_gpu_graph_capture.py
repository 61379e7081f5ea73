"""The replay step captured in a CUDA graph (as bench.py times it) gives the
eager results — with the sampler's in-kernel generator and with the Rng's
side-stream lookahead (a fork joined inside the captured region)."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _inputs(dev, steps, n, lmax, seed, start=1):
    g = np.random.default_rng(seed)
    out = []
    for _ in range(steps):
        toff = np.arange(0, (n + 1) * lmax, lmax, dtype=np.int64)
        b = dict(rollout_id=np.arange(start, start + n, dtype=np.int64),
                 reward=(g.random(n) < 0.5).astype(np.float64),
                 group_offsets=np.arange(0, n + 1, 8, dtype=np.int64), tok_offsets=toff,
                 tokens=g.integers(0, 1 << 30, n * lmax).astype(np.int32),
                 logp_old=(g.standard_normal(n * lmax) * 0.1 - 1).astype(np.float32))
        out.append({k: torch.from_numpy(v).to(dev) for k, v in b.items()})
        start += n
    return out


@pytest.mark.parametrize("lookahead", ["in-kernel", "side-stream"])
def test_captured_steps_match_eager(lookahead, monkeypatch):
    if not torch.cuda.is_available():
        pytest.fail("GPU test requested but CUDA is not available")
    from paper_2604_08706_b200 import Rng, ShardedReplayBuffer

    if lookahead == "side-stream":
        monkeypatch.setenv("RB_LOOKAHEAD_MIN_DRAWS", "0")
    dev = torch.device("cuda", 0)
    T, N, B, n, lmax, steps = 2, 256, 128, 64, 40, 4
    fill = _inputs(dev, 1, N, lmax, 1)[0]
    fill["group_offsets"] = torch.arange(0, N + 1, 8, dtype=torch.int64, device=dev)
    batches = _inputs(dev, steps + 1, n, lmax, 2, start=N + 1)  # [0]: eager warm-up
    results = []
    for mode in ("eager", "graph"):
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            buf = ShardedReplayBuffer(T, N, max_tokens=lmax)
            buf.set_stream(s.cuda_stream)
            rng = Rng(9).stream("buffer_sampling")
            buf.insert(**fill, assume_unique=True)
            tok = [torch.zeros(B * lmax + 8, dtype=torch.int32, device=dev) for _ in range(steps)]
            dl = [torch.zeros(B * lmax + 8, dtype=torch.float32, device=dev) for _ in range(steps)]
            lpn = torch.full((B * lmax + 8,), -1.05, dtype=torch.float32, device=dev)
            stats = torch.zeros(5, dtype=torch.float64, device=dev)
            buf.synchronize()

            def run(lo, hi):
                for i in range(lo, hi):
                    buf.insert(**batches[i + 1], assume_unique=True)
                    buf.sample_device(B, rng)
                    buf.gather(tok[i], None, None)
                    buf.loss_grpo(lpn, dl[i], 0.2, 0.28, stats=stats)

            # warm-up step (allocates the per-batch device buffers), as bench.py does
            buf.insert(**batches[0], assume_unique=True)
            buf.sample_device(B, rng)
            buf.gather(tok[0], None, None)
            buf.loss_grpo(lpn, dl[0], 0.2, 0.28, stats=stats)
            buf.synchronize()
            if mode == "eager":
                run(0, steps)
            else:
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=s, capture_error_mode="relaxed"):
                    run(0, steps)
                g.replay()
            torch.cuda.synchronize()
            results.append(([t.cpu().numpy() for t in tok], [d.cpu().numpy() for d in dl],
                            buf.dump()))
    (te, de, dump_e), (tg, dg, dump_g) = results
    for i in range(steps):
        assert np.array_equal(te[i], tg[i]), f"tokens differ at step {i}"
        assert np.array_equal(de[i], dg[i]), f"dlogp differs at step {i}"
    assert dump_e == dump_g
