"""``lbvh.cli`` -> paper_1908_11807_b200.cli (a real module so that
``python -m lbvh.cli`` works through the shim)."""

import sys

from paper_1908_11807_b200.cli import *  # noqa: F401,F403
from paper_1908_11807_b200.cli import main  # noqa: F401

if __name__ == "__main__":
    sys.exit(main())
