"""The INTEGRATION.md rebinding, exercised: device outcomes recorded on a
B200 (tests/golden/harness_outcomes.npz, made by make_harness_fixture.py)
are replayed through the reference's own, unmodified harness
(csvd.bench.run_benchmark, /root/reference/pkg/src/csvd/bench.py:317-404),
whose _validate_step (:224-265) checks every outcome against the dense
oracle; the run's outcome_sha256 must equal the reference's own run.

Needs the reference importable (this build container); skipped elsewhere."""
import os
import sys

import numpy as np
import pytest

REF = "/root/reference/pkg/src"
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
pytestmark = pytest.mark.skipif(not os.path.isdir(REF) or not os.path.exists(os.path.join(GOLD, "harness_outcomes.npz")),
                                reason="needs /root/reference and the recorded device outcomes")
KINDS = ("topk_exact", "softmax_eps", "topp_mass")
FBS = {-1: None, 0: "partial_expand", 1: "relax_eps", 2: "full_vocab"}


def _ref():
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import csvd
    import csvd.bench
    return csvd


def test_device_outcomes_pass_the_reference_harness(monkeypatch):
    csvd = _ref()
    from csvd.bench import BenchSpec
    from csvd.certify import CertStatus
    from csvd.cluster_index import load_index
    from csvd.decode import DecodeOutcome, StepMetrics
    z = np.load(os.path.join(GOLD, "harness_outcomes.npz"))
    n = len(z["ints"])
    spec = BenchSpec()
    table = csvd.synth_vocab(spec.vocab_size, spec.hidden_dim, spec.n_modes, spec.spread, spec.table_seed)
    index = load_index(os.path.join(GOLD, "harness_index.csvi"))
    cfg = spec.decode_config()
    step = {"t": 0}

    def replay(tbl, ix, h, c, k_max=None):  # what csvd.bench.decode_step = b200.decode_step returns
        t = step["t"]
        step["t"] += 1
        kind, fb, sub, opened, pops, fs, fbnd, k_eff = (int(x) for x in z["ints"][t])
        assert k_max == k_eff, "the harness's AdaptiveBudget trajectory differs from the recorded one"
        a, b = z["off"][t], z["off"][t + 1]
        eps, umax, kth, xi, rho = (float(x) for x in z["scal"][t])
        st = StepMetrics(sub_size=sub, ratio=sub / ix.vocab_size, clusters_opened=opened, xi=xi,
                         cert_kind=KINDS[kind], fallback=FBS[fb], rho=rho, flops_sparse=fs, flops_bounds=fbnd,
                         heap_pops=pops)
        return DecodeOutcome(token_ids=z["ids"][a:b].copy(), logits=z["logits"][a:b].copy(),
                             status=CertStatus(KINDS[kind], eps, umax, kth), fallback_used=FBS[fb], stats=st)

    ref_report = csvd.bench.run_benchmark(table, index, cfg, n, validate=False)
    monkeypatch.setattr(csvd.bench, "decode_step", replay)
    dev_report = csvd.bench.run_benchmark(table, index, cfg, n, validate=True)  # raises OracleViolation on failure
    assert dev_report.oracle["steps_validated"] == n
    assert dev_report.aggregates["outcome_sha256"] == ref_report.aggregates["outcome_sha256"]
