"""``python -m paper_2003_01836_b200 run|sweep|verify ...`` (the reference's ``bltc``)."""
from .cli import main

raise SystemExit(main())
