"""bench.py's CPU-side contract: the reference arm (the oracle, as it
stands) prints one JSON line with the required keys."""
import json
import sys


def test_reference_arm_json(monkeypatch, capsys):
    import bench
    monkeypatch.setattr(sys, "argv", ["bench.py", "--impl", "reference", "--steps", "2",
                                      "--warmup", "0", "--ref-planes", "4"])
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK"):
        monkeypatch.delenv(k, raising=False)
    bench.main()
    lines = [l for l in capsys.readouterr().out.splitlines() if l.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "dtype", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["rc"] == 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] == 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0
    assert d["cpu_baseline"]["available_cores"] >= 1 and d["cpu_baseline"]["cpu_model"]


def test_cpu_baseline_protocol():
    """cpu_baseline uses the reference arm's protocol (pinned core, same
    sample) and restores the process affinity afterwards."""
    import os
    import bench
    before = os.sched_getaffinity(0)
    d = bench.cpu_baseline_sample(steps=1, warmup=0)
    assert os.sched_getaffinity(0) == before
    assert d["kind"] == "oracle" and d["cores"] == 1 and d["value"] > 0
    assert d["pinned_core"] in before and d["available_cores"] == len(before)
    assert d["other_configs"]["C1_steps_per_s"] > 0 and d["other_configs"]["C3_steps_per_s"] > 0
    est = d["k_process_estimate"]
    assert est["kind"] == "estimate" and est["processes"] == len(before) and est["value"] > 0


def test_stale_ncu_numbers_are_not_reported(tmp_path, monkeypatch):
    """profiles/ncu_traffic.json entries count only for the sources they were
    captured from (kernel_src_sha16)."""
    import json as _json
    import bench
    p = tmp_path / "t.json"
    sha = bench.kernel_src_sha16()
    p.write_text(_json.dumps({"entries": {
        "fused_newton/contracted": {"dram_bytes": 1.0, "fp64_per_cell": 2.0, "src_sha16": sha, "source": "x"},
        "fused_newton/exact": {"dram_bytes": 3.0, "fp64_per_cell": 4.0, "src_sha16": "0" * 16, "source": "y"}}}))
    monkeypatch.setattr(bench, "TRAFFIC_JSON", str(p))
    e, state = bench.ncu_entry("fused_newton", "contracted")
    assert state == "current" and e["dram_bytes"] == 1.0
    e, state = bench.ncu_entry("fused_newton", "exact")
    assert e is None and state.startswith("stale")
    e, state = bench.ncu_entry("lu_solve", "composed")
    assert e is None and state == "missing"
