"""``python -m paper_2305_07030_b200`` -- the spec's command line (cli.py)."""
import sys

from .cli import main

sys.exit(main())
