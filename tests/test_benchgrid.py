"""Benchmark grid (benchgrid.py, mirror of the reference bench.py): CSV schema, resume keys and
the speedup report on CPU; one tiny fused-vs-baseline grid on the GPU."""

import csv

import pytest
import torch

from paper_2511_13645_b200 import benchgrid as bg


def _rows(path, rows):
    with open(path, "w", newline="") as fh:
        w = csv.DictWriter(fh, fieldnames=bg.CSV_COLUMNS)
        w.writeheader()
        for r in rows:
            w.writerow(r)


def _rec(variant, repeat, ms, pairs, peak):
    cfg = bg.BenchConfig(dataset="synth:powerlaw:N=100,deg=4,exp=2.1,seed=1", variant=variant, k1=5, k2=3,
                         batch=16, base_seeds=(42 + repeat,), steps=4, warmup=1, d_feat=8, hidden=8, classes=3)
    return bg.BenchRecord(cfg, repeat, 42 + repeat, ms, ms * 0.9, ms * 1.1, pairs, peak, "2026-01-01T00:00:00")


def test_report_medians_and_ratios(tmp_path):
    p = tmp_path / "grid.csv"
    rows = [_rec("baseline", 0, 2.0, 100.0, 4000).to_row(), _rec("baseline", 1, 4.0, 50.0, 6000).to_row(),
            _rec("fused", 0, 1.0, 200.0, 1000).to_row(), _rec("fused", 1, 1.0, 200.0, 1000).to_row()]
    _rows(p, rows)
    recs = bg.read_records(str(p))
    assert len(recs) == 4 and recs[0].key() == _rec("baseline", 0, 0, 0, 0).key()
    (s,) = bg.report_speedups(str(p))
    assert s["baseline_step_ms"] == 3.0 and s["fused_step_ms"] == 1.0 and s["step_speedup"] == 3.0
    assert s["pairs_speedup"] == 200.0 / 75.0 and s["mem_ratio"] == 5.0
    assert "3.00x" in bg.format_report([s])
    out = tmp_path / "summary.csv"
    bg.write_summary_csv([s], str(out))
    got = list(csv.DictReader(open(out)))
    assert list(got[0]) == bg.SUMMARY_COLUMNS and float(got[0]["mem_ratio"]) == 5.0


def test_reference_schema_first_and_reference_files_read(tmp_path):
    assert bg.CSV_COLUMNS[:len(bg.REF_COLUMNS)] == bg.REF_COLUMNS
    assert bg.CSV_COLUMNS[len(bg.REF_COLUMNS):] == ["seeds_per_s", "hbm_gbs_alg", "frac_hbm_peak", "draws_per_s",
                                                    "gpus", "alpha", "dtype", "cpu_cores"]
    # a file written with the reference's columns only (its own harness) still parses
    p = tmp_path / "ref.csv"
    with open(p, "w", newline="") as fh:
        w = csv.DictWriter(fh, fieldnames=bg.REF_COLUMNS)
        w.writeheader()
        for v in ("baseline", "fused"):
            row = _rec(v, 0, 2.0 if v == "baseline" else 1.0, 10.0, 8).to_row()
            w.writerow({c: row[c] for c in bg.REF_COLUMNS})
    recs = bg.read_records(str(p))
    assert [r.seeds_per_s for r in recs] == [None, None]
    (s,) = bg.report_speedups(str(p))
    assert s["step_speedup"] == 2.0 and s["fused_hbm_gbs_alg"] is None


def test_extra_columns_round_trip(tmp_path):
    r = _rec("fused", 0, 1.0, 5.0, 3)
    r.seeds_per_s, r.hbm_gbs_alg, r.frac_hbm_peak, r.draws_per_s = 1024.0, 900.5, 0.14, 3.5e10
    r.gpus, r.alpha, r.dtype, r.cpu_cores = 1, 2.1, "fp32", 16
    p = tmp_path / "g.csv"
    _rows(p, [r.to_row()])
    (back,) = bg.read_records(str(p))
    assert back.key() == r.key()
    assert (back.seeds_per_s, back.hbm_gbs_alg, back.frac_hbm_peak, back.draws_per_s) == (1024.0, 900.5, 0.14, 3.5e10)
    assert (back.gpus, back.alpha, back.dtype, back.cpu_cores) == (1, 2.1, "fp32", 16)


def test_schema_errors(tmp_path):
    p = tmp_path / "bad.csv"
    p.write_text("dataset,variant\nx,fused\n")
    with pytest.raises(ValueError, match="missing columns"):
        bg.read_records(str(p))
    row = _rec("fused", 0, 1.0, 1.0, 1).to_row()
    row["k1"] = "zero"
    _rows(p, [row])
    with pytest.raises(ValueError, match="row 2"):
        bg.read_records(str(p))
    _rows(p, [_rec("fused", 0, 1.0, 1.0, 1).to_row()])
    with pytest.raises(ValueError, match="missing baseline"):
        bg.report_speedups(str(p))
    with pytest.raises(ValueError, match="unknown variant"):
        bg.BenchConfig(dataset="d", variant="unfused", k1=1, k2=1, batch=1)


@pytest.mark.gpu
def test_tiny_grid_on_the_gpu(tmp_path):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    out = tmp_path / "grid.csv"
    spec = "synth:powerlaw:N=5000,deg=10,exp=2.1,seed=1"
    recs = bg.run_grid([spec], [(10, 5)], [256], ["fused", "baseline"], str(out), base_seeds=(42,), steps=3,
                       warmup=1, d_feat=32, hidden=16, classes=4, log=lambda m: None)
    assert len(recs) == 2
    again = bg.run_grid([spec], [(10, 5)], [256], ["fused", "baseline"], str(out), base_seeds=(42,), steps=3,
                        warmup=1, d_feat=32, hidden=16, classes=4, log=lambda m: None)
    assert again == []  # resumed: nothing left to run
    (s,) = bg.report_speedups(str(out))
    assert s["fused_step_ms"] > 0 and s["baseline_step_ms"] > 0
    assert s["baseline_peak_bytes"] > s["fused_peak_bytes"]  # the materialised blocks
    fused = [r for r in bg.read_records(str(out)) if r.config.variant == "fused"][0]
    assert fused.seeds_per_s > 0 and fused.hbm_gbs_alg > 0 and 0 < fused.frac_hbm_peak < 1
    assert fused.draws_per_s > 0 and fused.gpus == 1 and fused.alpha == 2.1 and fused.dtype == "fp32"
