"""``python -m paper_1608_04647_b200 fit-srm|bench ...`` (see cli.py)."""
import sys

from .cli import main

sys.exit(main())
