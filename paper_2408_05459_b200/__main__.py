"""`python -m paper_2408_05459_b200 run|gen|oracle` (reference: ancka/__main__.py)."""
import sys

from .cli import main

sys.exit(main())
