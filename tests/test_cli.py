"""CLI compatible with simtgraph-bench (pkg/tests/test_bench.py re-targeted).
Config errors need no GPU; runs and --verify are gpu tests."""

import csv

import numpy as np
import pytest

from paper_1002_4482_b200 import cli
from paper_1002_4482_b200.cli import COLUMNS, build_parser, main


def _read(path):
    with open(path, newline="") as f:
        return list(csv.DictReader(f))


def test_list_algorithms_reject_graph_families():
    assert main(["--algo", "wyllie", "--family", "tree", "--n", "100"]) == 2
    assert main(["--algo", "rs64", "--family", "random", "--n", "100"]) == 2


def test_rs48_thread_cap_is_a_config_error():
    assert main(["--algo", "rs48", "--threads", "65536", "--n", "100"]) == 2


def test_threads_and_blocks_are_exclusive():
    assert main(["--algo", "wyllie", "--n", "100", "--threads", "8", "--blocks", "2"]) == 2


def test_bad_numeric_flags():
    assert main(["--algo", "sv", "--n", "100", "--reps", "0"]) == 2
    assert main(["--algo", "sv", "--family", "random", "--density", "1.5", "--n", "100"]) == 2
    assert main(["--algo", "sv", "--n", "-3"]) == 2


def test_unknown_algorithm_rejected_by_parser():
    with pytest.raises(SystemExit) as e:
        main(["--algo", "quicksort", "--n", "10"])
    assert e.value.code == 2


def test_cpu_oracles_are_not_gpu_algorithms():
    assert main(["--algo", "seq_lr", "--n", "10"]) == 2
    assert main(["--algo", "seq_cc", "--n", "10"]) == 2


def test_env_var_supplies_default_seed(monkeypatch):
    monkeypatch.setenv(cli.SEED_ENV, "77")
    args = build_parser().parse_args(["--algo", "sv", "--n", "10"])
    assert args.seed == 77


def test_rank_check_is_complete():
    succ = np.array([3, 4, 2, 1, 2])
    assert cli._check_ranks(succ, np.array([4, 2, 0, 3, 1])) == -1
    assert cli._check_ranks(succ, np.array([4, 2, 0, 1, 3])) >= 0
    assert cli._check_ranks(succ, np.array([4, 2, 0, 3, 3])) >= 0


@pytest.mark.gpu
def test_csv_rows_and_aggregate(cuda, tmp_path):
    out = tmp_path / "b.csv"
    assert main(["--algo", "rs64", "--n", "5000", "--reps", "3", "--threads", "16", "--seed", "3",
                 "--out", str(out)]) == 0
    rows = _read(out)
    assert list(rows[0].keys()) == COLUMNS
    totals = [r for r in rows if r["kernel"] == "total" and r["rep"] != "agg"]
    aggs = [r for r in rows if r["rep"] == "agg"]
    assert len(totals) == 3 and len(aggs) == 1
    assert all(float(r["wall_time"]) > 0 for r in totals)
    assert all(r["max_sublist"] != "" for r in totals)


@pytest.mark.gpu
@pytest.mark.parametrize("algo,family", [("wyllie", "list"), ("rs48", "list"), ("rs64", "list"),
                                         ("rs_even", "list"), ("sv", "list"), ("sv", "tree"), ("sv", "random")])
def test_verify_passes(cuda, algo, family, capsys):
    n = "4096" if algo == "rs_even" else "3000"
    args = ["--algo", algo, "--family", family, "--n", n, "--reps", "2", "--verify", "--threads", "64"]
    if family == "random":
        args += ["--density", "0.002"]
    assert main(args) == 0
    assert "PASS" in capsys.readouterr().out


@pytest.mark.gpu
def test_verify_detects_corruption(cuda, monkeypatch, capsys):
    real = cli.run_algorithm

    def corrupt(*a, **k):
        out, st = real(*a, **k)
        out = np.array(out)
        out[7] += 1
        return out, st
    monkeypatch.setattr(cli, "run_algorithm", corrupt)
    assert main(["--algo", "rs64", "--n", "500", "--reps", "1", "--verify", "--threads", "16"]) == 1
    assert "FAIL" in capsys.readouterr().out


@pytest.mark.gpu
def test_plot_data(cuda, tmp_path):
    out, plot = tmp_path / "b.csv", tmp_path / "p.csv"
    assert main(["--algo", "wyllie", "--n", "2000", "--reps", "2", "--blocks", "1", "--blocks", "2",
                 "--out", str(out), "--plot-data", str(plot)]) == 0
    rows = _read(plot)
    assert len(rows) == 2 and float(rows[0]["speedup"]) == 1.0


def test_host_expectations_match_reference_examples():
    # test_core.py:46-59 known answers, and a labelling that merges two
    # components is caught (the host check is the component minimum)
    assert cli._host_ranks(np.array([1, 2, 2])).tolist() == [2, 1, 0]
    assert cli._host_ranks(np.array([3, 4, 2, 1, 2])).tolist() == [4, 2, 0, 3, 1]
    lab = cli._host_labels(6, np.array([[0, 3], [3, 5], [2, 4]]))
    assert lab.tolist() == [0, 1, 2, 0, 2, 0]
    from paper_1002_4482_b200.core import compare_arrays
    assert compare_arrays(lab, np.zeros(6, dtype=np.int64)) == 1
