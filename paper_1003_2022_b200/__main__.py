"""``python -m paper_1003_2022_b200 <subcommand>``: the command line (cli.py)."""

from .cli import main

raise SystemExit(main())
