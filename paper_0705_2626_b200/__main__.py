"""``python -m paper_0705_2626_b200 ...`` runs blockeig-bench (cli.py)."""

import sys

from .cli import main

sys.exit(main())
