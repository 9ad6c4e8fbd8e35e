"""The reference's self-check suite (checks.py:179-204) driving the CUDA ops."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_run_check_suite_passes_on_gpu():
    from paper_2507_04239_b200.checks import GPU_TOL, run_check_suite

    records = list(run_check_suite())
    assert records, "empty suite"
    kinds = {r["check"] for r in records}
    assert kinds == {"three_form", "vjp_chunked"}
    bad = [r for r in records if not r["passed"]]
    assert not bad, bad[:5]
    assert all(r["tol"] == GPU_TOL for r in records)
    # the p = 4 and odd-free normalized cases are all present
    assert {r["p"] for r in records if r["check"] == "three_form"} == {2, 4}
    assert any(r["normalized"] for r in records)


def test_check_records_are_json_lines():
    import json

    from paper_2507_04239_b200.checks import three_form_records

    recs = list(three_form_records(t_values=(5,), chunk_sizes=(2,), p_values=(2,), gating=(True,),
                                   normalize=(True,)))
    assert len(recs) == 1
    line = json.loads(json.dumps(recs[0]))
    assert set(line) == {"check", "p", "t", "c", "gated", "normalized", "max_rel_err", "tol", "seed",
                         "passed"}
    assert line["passed"] and np.isfinite(line["max_rel_err"])


def test_cli_bench_and_equiv(capsys):
    """cli.py bench / equiv records through the CUDA ops."""
    import json

    from paper_2507_04239_b200.cli import main

    assert main(["bench", "--t", "256", "--chunk", "64", "--heads", "2", "--gating",
                 "--repeats", "2", "--dtype", "f32"]) == 0
    rows = [json.loads(x) for x in capsys.readouterr().out.splitlines()]
    assert [r["config"]["form"] for r in rows] == ["attention", "chunked"]
    for r in rows:
        assert r["tokens_per_sec"] > 0 and np.isfinite(r["checksum"])
        assert set(r) == {"config", "tokens_per_sec", "wall_ns_total", "per_op_ns", "flops", "checksum"}
    assert abs(rows[0]["checksum"] - rows[1]["checksum"]) <= 1e-3 * max(1.0, abs(rows[0]["checksum"]))
    assert "power_full" in rows[1]["per_op_ns"]
    assert main(["equiv", "--format", "json", "--gating", "--normalize"]) == 0
    recs = [json.loads(x) for x in capsys.readouterr().out.splitlines()]
    assert all(r["max_rel_err"] <= 5e-3 for r in recs)
    assert main(["check", "--t", "8", "--chunk", "3", "--p", "2"]) == 0
