"""``python -m paper_1401_4068_b200`` -> the ente-compatible CLI (cli.py)."""
import sys

from .cli import main

sys.exit(main())
