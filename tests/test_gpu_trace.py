"""cfg-5 trace driver end to end on a short, tight trace: co-run engine (alloc -> prefill on
stream P || decode on stream D -> free), sampled oracle parity, bit-exact op-log replay."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_mla_trace_short_tight_pool():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "mla_trace.py"),
                        "--requests", "80", "--layers", "2", "--blocks", "200", "--samples", "4"],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert '"op_log_replay_tables_equal": true' in r.stdout


@pytest.mark.gpu
def test_mla_trace_short_expanded_prefill():
    """The same trace with the expanded-form MLA prefill (reading R32): the engine's prefill
    calls go through semipd_prefill_mla_expanded; sampled rows are checked against the oracle's
    expanded form (scripts/mla_trace.py exits non-zero on any parity miss)."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "mla_trace.py"),
                        "--requests", "80", "--layers", "2", "--blocks", "200", "--samples", "4",
                        "--expanded"],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert '"prefill_form": "expanded (R32)"' in r.stdout
    assert '"op_log_replay_tables_equal": true' in r.stdout
