"""``python -m paper_2305_11103_b200`` -> the CLI (cli.py)."""
import sys

from .cli import main

sys.exit(main())
