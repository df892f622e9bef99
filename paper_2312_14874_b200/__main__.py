"""``python -m paper_2312_14874_b200 <scan|verify|bench|sweep> ...`` (cli.py)."""

import sys

from .cli import main

sys.exit(main())
