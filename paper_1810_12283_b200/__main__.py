"""`python -m paper_1810_12283_b200 <subcommand> ...` — the gradkrig tools on the B200 path (cli.py)."""
import sys

from .cli import main

sys.exit(main())
