"""``python -m paper_2109_01232_b200 <solve|sweep-switch|sweep-restart|sweep-rhs|spmv-bench>``."""
import sys

from .cli import main

sys.exit(main())
