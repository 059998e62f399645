"""``python -m paper_2103_08825_b200 run|verify|plan`` (see cli.py)."""

import sys

from .cli import main

sys.exit(main())
