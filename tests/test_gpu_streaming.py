"""Batched tensor-core streaming (paper_2507_04239_b200.streaming): every
(batch, head) stream consumes its sequence step by step against a resident
state and must reproduce power_full on the whole sequence (reference
stream_chunk, chunked.py:416-458: "feeding chunks in order reproduces the
full-sequence chunked form").  Steps of mixed lengths, including ones that are
not a whole number of chunks (zero-padded inside the stream)."""

import numpy as np
import pytest
import torch

from oracle import power_oracle as O

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_2507_04239_b200")
from paper_2507_04239_b200 import streaming as S  # noqa: E402


def _inputs(b, t, h, seed, gated=True):
    q, k, v, g = O.generate_inputs(b, t, h, 64, 64, seed=seed, gating=gated)
    q, k, v = (torch.tensor(x).bfloat16().double().numpy() for x in (q, k, v))
    return q, k, v, g


def _stream(q, k, v, g, steps, normalize=False, chunk_size=None):
    dev = "cuda"
    Q, K, V = (torch.tensor(x, device=dev, dtype=torch.bfloat16) for x in (q, k, v))
    LG = None if g is None else torch.tensor(np.log(g), device=dev, dtype=torch.float32)
    state, ys, t0 = None, [], 0
    for n in steps:
        sl = slice(t0, t0 + n)
        y, state = S.stream_step(state, Q[:, sl], K[:, sl], V[:, sl], None if LG is None else LG[:, sl],
                                 normalize=normalize, chunk_size=chunk_size)
        ys.append(y)
        t0 += n
    return torch.cat(ys, 1).double().cpu().numpy(), state


@pytest.mark.parametrize("normalize", [False, True])
def test_steps_reproduce_the_whole_sequence(normalize):
    b, t, h = 2, 4096, 3
    q, k, v, g = _inputs(b, t, h, seed=81 + normalize)
    y, state = _stream(q, k, v, g, [1024, 1024, 512, 1536], normalize=normalize)
    y_ref, _ = O.chunked_forward(q, k, v, g, 2, 1024, normalize=normalize)
    err = O.max_rel_error(y, y_ref)
    print(f"streamed y vs oracle (normalize={normalize}): max_rel_error {err}")
    assert err <= 2e-2
    assert state.chunks == 1 + 1 + 1 + 2   # the 1536-token step is two chunks of 1024 (padded)


def test_end_state_matches_the_oracle_and_round_trips():
    """The resident state after the last step equals the whole sequence's end
    state S = sum_j (prod of later gates) phi(k_j) v_j^T in the reference's
    ChunkState layout, and converts back losslessly."""
    b, t, h = 1, 2048, 2
    q, k, v, g = _inputs(b, t, h, seed=91)
    _, state = _stream(q, k, v, g, [768, 1280])
    s, ks = state.to_chunk_states()
    K, V, G = (np.moveaxis(x, 2, 1).reshape(b * h, t, -1) for x in (k, v, g[..., None]))
    decay = np.concatenate([np.cumprod(G[:, ::-1, 0], axis=1)[:, ::-1][:, 1:], np.ones((b * h, 1))], axis=1)
    s_ref, ks_ref = O.update_state(K, V, decay, 2)
    s_ref, ks_ref = s_ref.reshape(b, h, *s_ref.shape[1:]), ks_ref.reshape(b, h, -1)
    es = float(np.linalg.norm(s - s_ref) / np.linalg.norm(s_ref))
    ek = float(np.linalg.norm(ks - ks_ref) / np.linalg.norm(ks_ref))
    print(f"end state vs oracle: norm-wise {es}, key_sum {ek}")
    assert es <= 1e-2 and ek <= 1e-2
    back = S.StreamState.from_chunk_states(s, ks, state.chunks, "cuda")
    assert torch.allclose(back.data, state.data, rtol=1e-6, atol=1e-6)


def test_resume_from_a_reference_state():
    """Start a stream from a ChunkState (here: the oracle's state after the
    first half) and the second half's outputs equal the whole-sequence ones."""
    b, t, h = 1, 2048, 2
    q, k, v, g = _inputs(b, t, h, seed=95)
    y_full, st_full = _stream(q, k, v, g, [1024, 1024])
    _, st_half = _stream(q[:, :1024], k[:, :1024], v[:, :1024], g[:, :1024], [1024])
    s, ks = st_half.to_chunk_states()
    resumed = S.StreamState.from_chunk_states(s, ks, st_half.chunks, "cuda")
    dev = "cuda"
    Q, K, V = (torch.tensor(x[:, 1024:], device=dev, dtype=torch.bfloat16) for x in (q, k, v))
    y2, _ = S.stream_step(resumed, Q, K, V, torch.tensor(np.log(g[:, 1024:]), device=dev, dtype=torch.float32))
    err = O.max_rel_error(y2.double().cpu().numpy(), y_full[:, 1024:])
    assert err <= 1e-2, err
