"""The driver's smoke() entry point as a GPU test: one small bf16 forward +
backward through torch autograd (the backward runs on autograd's worker
thread, which is where the tensor-map context binding once failed)."""

import pytest

pytestmark = pytest.mark.gpu


def test_graft_smoke():
    import __graft_entry__

    __graft_entry__.smoke()
