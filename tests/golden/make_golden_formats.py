"""Reference-written format fixtures (cli.py:71-83 write_csv, :131-135 _cache_store):

    python tests/golden/make_golden_formats.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
from levyh import cli as CLI  # noqa: E402
from tests import test_formats as T  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
CLI.write_csv(os.path.join(OUT, "formats_ref.csv"), T.HEADER, T.ROWS, T.META)
CLI._cache_store(os.path.join(OUT, "formats_cache"), "frac1d|s=0.5|N=4095|T=1.0", np.arange(5.0) / 7)
print(open(os.path.join(OUT, "formats_ref.csv")).read())
