"""``python -m paper_2107_02671_b200 ...`` runs the experiment CLI (cli.py)."""

import sys

from .cli import main

sys.exit(main())
