"""python -m paper_2010_00626_b200 <subcommand>: the CLI mirror (cli.py)."""

import sys

from .cli import main

sys.exit(main())
