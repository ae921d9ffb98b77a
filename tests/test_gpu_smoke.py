"""The driver's smoke() entry point must keep working as layouts evolve."""

import pytest

pytestmark = pytest.mark.gpu


def test_graft_entry_smoke(cuda):
    import __graft_entry__

    __graft_entry__.smoke()
