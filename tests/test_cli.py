"""The GPU CLI front-end (paper_2203_00854_b200/cli.py) against the reference CLI's own
tests (tests/test_cli.py:32-75 of the reference): envelope, commvolume reference points,
exit codes, and - on the GPU - simulate's measured ledger equal to predict_block_ledger."""
import json

import pytest

from paper_2203_00854_b200.cli import EXIT_CONSTRAINT, EXIT_OK, EXIT_USAGE, main


def _run(capsys, *argv):
    code = main(list(argv))
    cap = capsys.readouterr()
    return code, cap.out, cap.err


def test_commvolume_reference_point(capsys):
    code, out, _ = _run(capsys, "--no-timestamp", "commvolume", "--k", "1", "--devices", "4", "--heads", "4")
    assert code == EXIT_OK
    doc = json.loads(out)
    assert doc["schema"] == "evoplan-cli-v1" and doc["command"] == "commvolume" and "timestamp" not in doc
    assert doc["result"]["tp_volume"] == 18.0
    assert doc["result"]["dap_volume"] == 4.5


def test_commvolume_single_device_zero(capsys):
    code, out, _ = _run(capsys, "--no-timestamp", "commvolume", "--k", "1", "--devices", "1")
    assert code == EXIT_OK
    result = json.loads(out)["result"]
    assert result["tp_volume"] == 0.0 and result["dap_volume"] == 0.0


def test_commvolume_head_limit_exit_code(capsys):
    code, _, err = _run(capsys, "--no-timestamp", "commvolume", "--k", "1", "--devices", "8", "--heads", "4")
    assert code == EXIT_CONSTRAINT
    assert "head-count" in json.loads(err)["error"]


def test_commvolume_matches_reference_model():
    """the closed form equals the reference model's at a grid of points (golden values
    computed from commcost.py:70-123: 24K(N-1)/N and 3K(N-1)/N + 12K(N-1)/N^2)"""
    from paper_2203_00854_b200.commcost import CommModel
    for k in (0.5, 1.0, 3.0):
        for n in (1, 2, 4, 8):
            r = CommModel(n_heads=8).compare(k, n)
            assert r.tp_volume == pytest.approx(24 * k * (n - 1) / n)
            assert r.dap_volume == pytest.approx(3 * k * (n - 1) / n + 12 * k * (n - 1) / n ** 2)


def test_simulate_indivisible_extent_is_usage_error(capsys):
    code, _, err = _run(capsys, "--no-timestamp", "simulate", "--devices", "3", "--n-seq", "8", "--n-res", "16")
    assert code == EXIT_USAGE
    assert "devices" in json.loads(err)["error"]


def test_bad_arguments_are_usage_errors(capsys):
    assert _run(capsys, "simulate")[0] == EXIT_USAGE  # --devices missing
    assert _run(capsys, "nonsense")[0] == EXIT_USAGE


@pytest.mark.gpu
@pytest.mark.parametrize("devices", [2, 4])
def test_simulate_matches_prediction_gpu(capsys, devices):
    code, out, _ = _run(capsys, "--no-timestamp", "simulate", "--devices", str(devices), "--seed", "31")
    assert code == EXIT_OK
    result = json.loads(out)["result"]
    assert result["rel_error"] <= result["rel_tolerance"]
    assert result["ledger_matches_prediction"] is True
    assert result["ledger"]["all_to_all"]["count"] == 6
    assert result["ledger"]["all_gather"]["count"] == 3
