"""``python -m paper_2510_11023_b200 ...``: the parafrac-compatible CLI (``cli.py``)."""

import sys

from .cli import main

sys.exit(main())
