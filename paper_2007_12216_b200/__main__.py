"""``python -m paper_2007_12216_b200 {verify,bench}`` (see cli.py)."""
import sys

from .cli import main

sys.exit(main())
