"""Run the REFERENCE's own CLI (gemmforge bench / verify) with the B200 engine
registered as variant "b200".

  python tools/run_gemmforge_b200.py verify --alg b200
  python tools/run_gemmforge_b200.py bench --alg goto,b200 --min 256 --max 1024 --step 256 --check

Needs the reference package (oracle/_ref, built by oracle/build_ref.sh, or any
importable `gemmforge`).
"""
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "oracle", "_ref"))

import gemmforge  # noqa: E402  (the reference)
from gemmforge import cli  # noqa: E402

from paper_1609_00076_b200 import register  # noqa: E402

register(gemmforge.registry.default_registry())
sys.exit(cli.main())
