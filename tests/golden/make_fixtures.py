"""Copies the reference's data fixtures (scenario files and the example
acceptance trace, /root/reference/proj/fixtures) into
tests/golden/reference_fixtures/ so the parity tests can use them where
/root/reference does not exist (the GPU box).  Data only, no source.  Run
in the build container:

    python tests/golden/make_fixtures.py
"""

import os
import shutil

SRC = "/root/reference/proj/fixtures"
DST = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_fixtures")

if __name__ == "__main__":
    os.makedirs(DST, exist_ok=True)
    for name in sorted(os.listdir(SRC)):
        shutil.copyfile(os.path.join(SRC, name), os.path.join(DST, name))
        print("copied", name)
