"""``python -m paper_2605_29291_b200 solve|gap ...`` (cli.py:374-389)."""
import sys

from .cli import main

sys.exit(main())
