"""``python -m paper_2110_08389_b200 <command> ...`` -- see cli.py."""
import sys

from .cli import main

sys.exit(main())
