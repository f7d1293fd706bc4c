"""CLI drop-in (reference cli.py:281-424): usage errors exit 2 before any device work (CPU);
the solve / convergence runs themselves are in tests/ref_suite/test_cli_solve.py (GPU)."""

import pytest

from paper_1512_06025_b200.cli import main


@pytest.mark.parametrize("argv", [["convergence", "--n", "1", "--meshes", "2"], ["solve", "--n", "1,2"],
                                  ["solve", "--n", ""], ["bogus"]])
def test_usage_errors_exit_2(tmp_path, argv):
    with pytest.raises(SystemExit) as exc:
        main(argv + ["--out", str(tmp_path)] if argv[0] != "bogus" else argv)
    assert exc.value.code == 2


def test_diagnostics_are_out_of_scope(tmp_path):
    assert main(["ops", "--n", "1..2"]) == 2
    assert main(["check"]) == 2
