"""Host-side checks of the batched streaming module (no GPU)."""

import numpy as np
import pytest
import torch

from oracle import power_oracle as O
from paper_2507_04239_b200 import streaming as S
from paper_2507_04239_b200.errors import InvalidSpec


def test_slot_map_is_a_bijection_onto_the_ndmi_features():
    feat, slots, omega = S._slot_features()
    idx, w = O.ndmi_table(2, 64)
    assert len(feat) == len(idx) == 2080
    assert sorted(feat.tolist()) == list(range(2080))
    # omega = w^2 of the matching NDMI feature (1 on the diagonal, 2 off it)
    np.testing.assert_allclose(omega, w[feat] ** 2)


def test_state_conversion_round_trip_on_cpu():
    rng = np.random.default_rng(3)
    s = rng.standard_normal((1, 2, 2080, 64))
    ks = rng.standard_normal((1, 2, 2080))
    st = S.StreamState.from_chunk_states(s, ks, 4, "cpu")
    s2, ks2 = st.to_chunk_states()
    np.testing.assert_allclose(s2, s, rtol=1e-6, atol=1e-6)
    np.testing.assert_allclose(ks2, ks, rtol=1e-6, atol=1e-6)


def test_rejects_shapes_outside_the_tensor_core_path():
    x = torch.zeros(1, 128, 1, 32)
    with pytest.raises(InvalidSpec):
        S.stream_step(None, x, x, x, p=2)
    y = torch.zeros(1, 128, 1, 64)
    with pytest.raises(InvalidSpec):
        S.stream_step(None, y, y, y, p=4)
