"""apply_filter's grouped degree schedule (cf_degree_schedule), host-only."""
import pytest

import paper_1803_02156_b200 as cf
from paper_1803_02156_b200.kernels import degree_schedule


@pytest.mark.parametrize("np_", [2, 3, 4, 5, 6, 7, 11, 12, 13, 500])
def test_degree_schedule_covers_every_degree_once(np_):
    fc = cf.filter_coefficients(-0.3, 0.3, cf.spectral_map(-7.0, 7.0, 0.01), np_)
    sched = degree_schedule(fc)
    assert [d[0] for d in sched] == list(range(3, np_ + 1))
    gcoef = lambda q: fc.g[q] * fc.c[q]  # noqa: E731
    # every degree's g_p c_p enters X exactly once, at the step that closes its group
    seen = []
    pending = []
    for p, kind, gw, gu, gc in sched:
        pending.append(p)
        if kind == 1:
            assert gw == gu == gc == 0.0
            continue
        grp = {0: 1, 2: 2, 3: 3}[kind]
        assert pending[-grp:] == list(range(p - grp + 1, p + 1)) and len(pending) == grp
        coefs = {0: [gc], 2: [gu, gc], 3: [gw, gu, gc]}[kind]
        assert coefs == [gcoef(q) for q in pending]
        seen += pending
        pending = []
    assert not pending and seen == list(range(3, np_ + 1))
    if np_ >= 5:
        assert sum(1 for d in sched if d[1] == 3) == (np_ - 2) // 3
