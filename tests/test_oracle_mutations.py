"""Every plausible oracle mistake listed in tools/oracle_mutations.py (the four the
round-1 review found unpinned among them) must make tests/test_oracle_pins.py fail."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.slow
def test_no_oracle_mutation_survives_the_pins():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "oracle_mutations.py")],
                       capture_output=True, text=True, timeout=1500)
    assert r.returncode == 0, r.stdout + r.stderr
