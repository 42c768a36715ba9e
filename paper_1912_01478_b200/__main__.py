"""python -m paper_1912_01478_b200 -> the CLI (cli.py)."""
import sys

from .cli import main

sys.exit(main())
