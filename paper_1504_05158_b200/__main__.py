"""``python -m paper_1504_05158_b200 solve|validate|sweep ...`` (cli.py)."""
import sys

from .cli import main

sys.exit(main())
