"""The scaling report (paper_1806_08741_b200/scaling.py)
against the unmodified reference's bench.hpp analysis: the same alpha,
speedups and efficiencies bit for bit and byte-identical CSV and markdown
(first column renamed from Threads to GPUs), on random timing records with
and without a connectivity series; plus the reference suite's analytic
anchors and the CSV round trip."""
import numpy as np
import pytest

from paper_1806_08741_b200 import scaling as sc


def test_matches_reference(reference_lib):
    rng = np.random.default_rng(21)
    for trial in range(30):
        ps = [1, 2, 4, 8][: int(rng.integers(2, 5))]
        both = trial % 3 == 0
        recs = []
        for conn in ([False, True] if both else [False]):
            t1 = float(rng.uniform(0.5, 50.0))
            for p in ps:
                recs.append(sc.TimingRecord(p, t1 / p * float(rng.uniform(1.0, 1.6)), conn))
        ours = sc.make_report(recs)
        alpha, sp, ef, csv, md = reference_lib.scaling_report(
            [r.workers for r in recs], [r.time_seconds for r in recs],
            [int(r.with_connectivity) for r in recs])
        assert ours.alpha == alpha
        assert ours.speedups == list(sp) and ours.efficiencies == list(ef)
        assert sc.emit_scaling_csv(ours) == csv
        assert sc.emit_scaling_markdown(ours, unit="Threads") == md
        back = sc.parse_scaling_csv(csv)
        assert back.alpha == ours.alpha and back.records == ours.records


def test_analytic_anchors(reference_lib):
    for alpha in (0.0, 0.05, 0.3, 1.0):
        for p in (1, 2, 8, 64):
            assert sc.amdahl_bound(alpha, p) == reference_lib.lib.ref_amdahl_bound(alpha, p)
            assert (sc.amdahl_efficiency_bound(alpha, p)
                    == reference_lib.lib.ref_amdahl_efficiency_bound(alpha, p))
    # perfect scaling fits alpha = 0; flat times fit alpha = 1
    assert sc.fit_alpha([sc.TimingRecord(p, 8.0 / p) for p in (1, 2, 4, 8)]) == 0.0
    assert sc.fit_alpha([sc.TimingRecord(p, 8.0) for p in (1, 2, 4, 8)]) == 1.0
    with pytest.raises(ValueError):
        sc.fit_alpha([sc.TimingRecord(2, 1.0)])
    assert sc.make_report([sc.TimingRecord(1, 3.0)]).alpha == 1.0
