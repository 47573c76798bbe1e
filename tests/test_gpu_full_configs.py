"""Full-size configs 2 and 4 on the device (config 3 is run by
tools/config_runs.py, profiles/r1/configs_c3_c1.json): corpus generated in
HBM, index built on the device, the whole query batch run, and parity with
the CPU oracle checked through properties that need no oracle-sized build:
widths sized by the oracle's size_filter, sampled documents' term counts and
complete bit columns, sampled queries' l / skipped / hit lists."""
import os

import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.skipif(os.environ.get("COBS_SKIP_FULL_CONFIGS") == "1", reason="disabled")
@pytest.mark.parametrize("name", ["c4", "c2"])
def test_full_config_properties(gpu, name):
    from tools.config_runs import run
    r = run(name, n_sample_docs=3, n_sample_queries=20)
    checks = r["checks"]
    for key, ok in checks.items():
        if isinstance(ok, bool):
            assert ok, (name, key, r)
    assert r["query"]["n_queries"] == {"c2": 10_000, "c4": 50_000}[name]
