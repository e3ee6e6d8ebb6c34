"""``python -m paper_0910_4711_b200`` -> the ``vq`` command line (cli.py)."""
import sys

from .cli import main

sys.exit(main())
