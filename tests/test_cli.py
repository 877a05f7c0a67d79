"""Command line (cli.py of the reference): same commands,
flags and JSONL RunReport records, GPU underneath."""
import json
from pathlib import Path

import numpy as np
import pytest

import paper_2503_04422_b200 as P
from paper_2503_04422_b200 import cli

GOLD = Path(__file__).resolve().parent / "golden" / "pdx"


def test_gen_and_parser(tmp_path):
    out = tmp_path / "x.fvecs"
    assert cli.main(["gen", "--n", "50", "--d", "6", "--distribution", "skewed", "--seed", "3",
                     "--out", str(out)]) == 0
    np.testing.assert_array_equal(P.read_fvecs(out).data,
                                  P.gen_synthetic(50, 6, "skewed", 3).data)
    with pytest.raises(SystemExit):
        cli.build_parser().parse_args(["query", "--dataset", "a.pdx"])  # --queries missing
    args = cli.build_parser().parse_args(["sweep", "--dataset", "a", "--queries", "b",
                                          "--pruner", "bsa", "--selection-fractions", "0.1",
                                          "0.3"])
    assert args.pruner == "bsa" and args.selection_fractions == [0.1, 0.3]


def test_errors_become_system_exit(tmp_path):
    with pytest.raises(SystemExit, match="missing.pdx"):
        cli.main(["query", "--dataset", str(tmp_path / "missing.pdx"), "--queries", "q.fvecs"])
    (tmp_path / "bad.fvecs").write_bytes(b"\x01\x00")
    with pytest.raises(SystemExit, match="truncated"):
        cli.main(["convert", "--dataset", str(tmp_path / "bad.fvecs"),
                  "--out", str(tmp_path / "o.pdx")])


@pytest.mark.gpu
def test_convert_reproduces_reference_bytes(tmp_path):
    """gen + convert write the bytes the reference's convert wrote
    (tests/golden/make_pdx_golden.py: same seed, same collection)."""
    x = tmp_path / "x.fvecs"
    cli.main(["gen", "--n", "130", "--d", "8", "--seed", "2", "--out", str(x)])
    out = tmp_path / "x.pdx"
    cli.main(["convert", "--dataset", str(x), "--block-size", "64", "--out", str(out)])
    assert out.read_bytes() == (GOLD / "flat64.pdx").read_bytes()
    back = tmp_path / "back.fvecs"
    cli.main(["convert", "--dataset", str(out), "--out", str(back)])
    assert back.read_bytes() == x.read_bytes()


@pytest.mark.gpu
def test_query_and_sweep_end_to_end(tmp_path):
    data, q = tmp_path / "d.fvecs", tmp_path / "q.fvecs"
    cli.main(["gen", "--n", "20000", "--d", "32", "--distribution", "clustered",
              "--clusters", "64", "--seed", "1", "--out", str(data)])
    cli.main(["gen", "--n", "100", "--d", "32", "--distribution", "clustered",
              "--clusters", "64", "--seed", "1", "--out", str(q)])
    gt = tmp_path / "gt.ivecs"
    cli.main(["ground-truth", "--dataset", str(data), "--queries", str(q), "--out", str(gt)])
    flat = tmp_path / "flat.pdx"
    cli.main(["convert", "--dataset", str(data), "--out", str(flat)])
    rep = tmp_path / "flat.jsonl"
    cli.main(["query", "--dataset", str(flat), "--queries", str(q), "--pruner", "bond",
              "--criteria", "dmeans", "--ground-truth", str(gt), "--out", str(rep)])
    r = json.loads(rep.read_text())
    assert r["recall_mean"] == 1.0 and r["qps"] > 0
    assert set(r) == {"config", "recall_mean", "qps", "pruning_power", "phase_seconds",
                      "total_seconds"}
    assert 0 < r["pruning_power"]["mean"] < 1
    for pruner, floor in (("ads", 0.95), ("bsa", 0.95), ("bond", 1.0)):
        ivf = tmp_path / f"ivf_{pruner}.pdx"
        cli.main(["build-ivf", "--dataset", str(data), "--nlist", "32", "--pruner", pruner,
                  "--out", str(ivf)])
        out = tmp_path / f"{pruner}.jsonl"
        cli.main(["query", "--dataset", str(ivf), "--queries", str(q), "--pruner", pruner,
                  "--nprobe", "32", "--ground-truth", str(gt), "--out", str(out)])
        r = json.loads(out.read_text())
        assert r["recall_mean"] >= floor, (pruner, r)
        assert {"find_nearest_buckets", "distance_calculation",
                "query_preprocessing"} <= set(r["phase_seconds"])
    sw = tmp_path / "sweep.jsonl"
    cli.main(["sweep", "--dataset", str(tmp_path / "ivf_bond.pdx"), "--queries", str(q),
              "--pruner", "bond", "--selection-fractions", "0.1", "0.5", "--ground-truth",
              str(gt), "--out", str(sw)])
    recs = [json.loads(line) for line in sw.read_text().splitlines()]
    assert [r["config"]["nprobe"] for r in recs] == [n for n in (1, 2, 4, 8, 16, 32)
                                                     for _ in range(2)]
    assert recs[-1]["recall_mean"] == 1.0
