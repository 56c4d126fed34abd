"""python -m paper_2302_13431_b200 estimate ... (see cli.py)."""
import sys

from .cli import main

sys.exit(main())
