"""Write the I/O fixtures with the REFERENCE package (run in the build container only).

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/nb python tests/golden/make_io_golden.py

Produces tests/golden/io_ref.bin / io_ref.csv (ente.io_formats.save_ensemble,
/root/reference/pkg/src/ente/io_formats.py:23-34) for a small seeded ensemble,
and io_ref_results.json (write_results, io_formats.py:135-166, no timestamp)
for a fixed TEResult, so the drop-in's readers and writers are pinned to the
reference's bytes.
"""
import os

import numpy as np

from ente import io_formats
from ente.data import AnalysisConfig, EnsembleSeries, TEResult

HERE = os.path.dirname(os.path.abspath(__file__))
vals = np.random.default_rng(7).standard_normal((3, 5))
series = EnsembleSeries("chan-α", vals)
io_formats.save_ensemble(series, os.path.join(HERE, "io_ref.bin"), "bin")
io_formats.save_ensemble(series, os.path.join(HERE, "io_ref.csv"), "csv")
res = TEResult(source="X", target="Y", window=(10, 20), u_selected=3, te_value=0.125,
               surrogate_values=np.array([0.01, 0.02, 0.5]), p_value=1 / 3, significant=False,
               significant_corrected=False, te_minus_median_surrogate=0.105,
               te_curve=[(1, 0.1), (3, 0.125)])
cfg = AnalysisConfig(u_candidates=(1, 3), window=(10, 20), k=4, n_surrogates=3, seed=5)
io_formats.write_results([res], os.path.join(HERE, "io_ref_results.json"), cfg, timestamp=False)
print("wrote io fixtures")
