"""`python -m ndgauss ...` -- the reference console script `ndgauss` (pkg/pyproject.toml:15-16)."""
import sys

from paper_2405_20067_b200.cli import main

sys.exit(main())
