"""The C++ drop-in (include/gpudvfs_b200/gpu_api.hpp) against the reference's
own production path: integration/facade_test runs fit -> model files ->
clusters -> make_model_predictor -> schedule_d_dvfs through both and requires
identical decisions for all 16 SchedulerOptions combinations (plus predict
and the column-mismatch message).  Variants: a catalog profiled at every other
clock (general per-candidate kernel) or at three clocks per app ((app,
record) virtual apps on the partial-evaluation path), single device or a
gd_multi device group; every workload carries duplicate app_ids whose
default profiles differ."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
EXE = ROOT / "integration" / "_build" / "facade_test"


@pytest.mark.gpu
@pytest.mark.parametrize("args", [(), ("60", "8", "300"), ("60", "8", "300", "25"), ("40", "6", "200", "2", "1"),
                                  ("40", "6", "200", "25", "1")])
def test_facade_dropin_identical_to_reference(args):
    if not EXE.exists():
        pytest.skip("integration/_build/facade_test not built (make -C integration needs the reference headers)")
    r = subprocess.run([str(EXE), *args], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "FACADE OK" in r.stdout and " 0 mismatches" in r.stdout
