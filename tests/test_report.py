"""The `bench-adjoint` report (schema sinktail-report/1, proj/tools/sinktail_main.cpp:315-380) on the
device path: schema fields, plan-byte ledger, mode agreement and the pass rule."""
import json

import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_bench_adjoint_report(tmp_path, dtype):
    from paper_2605_08123_b200 import report
    out = tmp_path / "bench.json"
    r = report.bench_adjoint(seq_lens=(256, 640), half_band=128, head_dim=64, base_depth=10, epsilon=1.0,
                             repetitions=3, warmup=1, dtype=dtype, out_path=str(out))
    assert json.loads(out.read_text()) == r
    assert r["schema"] == "sinktail-report/1" and r["config"]["command"] == "bench-adjoint"
    for row in r["results"]:
        assert row["direct_plan_bytes"] == 4 * row["one_reference_plan_bytes"]
        L, w = row["L"], 128
        assert row["one_reference_plan_bytes"] == (L * (2 * w + 1) - w * (w + 1)) * (4 if dtype == "f32" else 2)
        assert row["max_abs_dQ"] <= row["grad_tolerance_rel_to_max"] * 10  # modes agree (relative to O(1) grads)
        assert row["speedup"] > 0 and row["one_reference_ms"]["min"] > 0
    assert isinstance(r["pass"], bool)
