"""`python -m paper_1510_08094_b200 ...`: the command-line front end (cli.py)."""
import sys

from .cli import main

sys.exit(main())
