"""The reference's acceptance gate (proj/tests/acceptance/acceptance_main.cpp)
compiled UNCHANGED against the drop-in headers (include/glu) and linked with
lib/libglu.so, i.e. every hot-path call runs on the B200 (oracle/Makefile
target `acceptance`; the binary travels with the tree).

Runnable here: criteria 3 (joint optimisation monotone over 50 seeded images,
rejected trials roll back bitwise; acceptance_main.cpp:104-145), 4 (thin-line
recovery at 1024^2 / s = 16; 148-162), 5 (exact <= fast <= gnu dominance chain
over 10,000 instances; 166-192), 7 (JBU collapses onto GNU; 249-262), 8 (metric
oracles; 264-290) and 9 (GLUP round trip and corruption names; 292-373).
Blocked: 1, 2 and 6 need the corpus photo tests/data/astronaut.png (absent,
not to be recreated) and 10 needs the CLI (out of scope) -- they report FAIL
with an IoError from the shim and are asserted to be exactly those four.
"""
import os
import re
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
RUNNABLE = {3, 4, 5, 7, 8, 9}
BLOCKED = {1, 2, 6, 10}


def test_reference_acceptance_gate_against_dropin(glu):
    exe = os.path.join(ROOT, "oracle", "_ref", "acceptance_b200")
    if not os.path.exists(exe):
        if not os.path.isdir("/root/reference/proj/tests/acceptance"):
            pytest.skip("acceptance_b200 not built and /root/reference absent")
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "acceptance"],
                       check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=900)
    print(r.stdout)
    res = {int(m.group(2)): (m.group(1), m.group(3))
           for m in re.finditer(r"\[(PASS|FAIL)\] criterion\s+(\d+): (.*)", r.stdout)}
    assert set(res) == RUNNABLE | BLOCKED, r.stdout + r.stderr
    for c in sorted(RUNNABLE):
        assert res[c][0] == "PASS", (c, res[c][1])
    for c in sorted(BLOCKED):
        assert res[c][0] == "FAIL" and "image I/O is not part of this build" in res[c][1], \
            (c, res[c][1])
    assert r.returncode == len(BLOCKED)
