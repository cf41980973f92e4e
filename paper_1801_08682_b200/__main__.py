"""``python -m paper_1801_08682_b200 run|convergence ...`` (src/__main__.py)."""
import sys

from .cli import main

sys.exit(main())
