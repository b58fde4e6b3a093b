"""``python -m paper_2403_06348_b200 <command> ...`` runs the CLI (cli.py)."""

import sys

from .cli import main

sys.exit(main())
