"""python -m paper_1301_4438_b200 ... (see cli.py)."""
import sys

from .cli import main

sys.exit(main())
