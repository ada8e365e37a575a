"""CPU: bench.py --impl reference runs the unmodified reference build (oracle/_ref) on the
host cores with the same config object as the GPU arm, and never maps this repo's product
library (the driver records which .so files the reference-arm process loaded)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

@pytest.mark.timeout(600)
@pytest.mark.parametrize("config", ["c1"])
def test_reference_arm_does_not_load_the_product(config):
    if not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libuniprefill_ref.so")):
        pytest.skip("oracle/_ref (the reference build) is not built")
    code = (
        "import sys, runpy\n"
        f"sys.argv = ['bench.py', '--impl', 'reference', '--config', '{config}', '--steps', '1', '--warmup', '0']\n"
        f"sys.path.insert(0, {ROOT!r})\n"
        f"runpy.run_path({os.path.join(ROOT, 'bench.py')!r}, run_name='__main__')\n"
        "maps = open('/proc/self/maps').read()\n"
        "print('PRODUCT_MAPPED', 'libuniprefill_b200' in maps, any(m.startswith('paper_2605_06221_b200') "
        "for m in sys.modules))\n")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=580, cwd=ROOT,
                         env=dict(os.environ, CUDA_VISIBLE_DEVICES=""))
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "tokens/s"
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1
    assert d["cpu_baseline"]["single_core"]["cores"] == 1 and d["cpu_baseline"]["nproc"] >= 1
    assert d["e2e"] == {"value": d["value"], "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert "PRODUCT_MAPPED False False" in out.stdout
