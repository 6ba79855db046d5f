"""the oracle under AddressSanitizer + UndefinedBehaviorSanitizer.

tests/harness/oracle_sanitize.c is compiled together with oracle/slo_oracle.c (-fsanitize=address,undefined,
-fno-sanitize-recover so any finding fails the run) and drives the oracle over every arrival kind, both batching
modes, speculation, warmup and the stop rule.  The test passes iff the driver exits 0 with its "ok" line."""
import os
import shutil
import subprocess

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)


@pytest.mark.skipif(shutil.which("gcc") is None, reason="gcc not available")
def test_oracle_clean_under_asan_ubsan(tmp_path):
    exe = tmp_path / "oracle_sanitize"
    cmd = ["gcc", "-O1", "-g", "-std=c11", "-fsanitize=address,undefined", "-fno-sanitize-recover=all",
           "-fno-omit-frame-pointer", "-o", str(exe), os.path.join(HERE, "harness", "oracle_sanitize.c"),
           os.path.join(ROOT, "oracle", "slo_oracle.c"), "-lm"]
    subprocess.check_call(cmd)
    env = dict(os.environ, ASAN_OPTIONS="detect_leaks=1:abort_on_error=0", UBSAN_OPTIONS="print_stacktrace=1")
    r = subprocess.run([str(exe)], capture_output=True, text=True, env=env, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert "oracle sanitize ok" in r.stdout, r.stdout
