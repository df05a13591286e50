"""Pin of the device's adj = (i*f + j)/f^2 (Alg. 2): the bucket sort
computes it as q0 = g * RN(1/f^2), q = fma(fma(-q0, f^2, g), RN(1/f^2), q0)
instead of a division. This checks, exhaustively over every fan-out
f in [2, 1024] and every sub-bucket g < f^2 (358M cases), that the formula
equals the correctly rounded IEEE quotient g / f^2 that the oracle uses."""
import os
import subprocess


def test_fma_refined_division_is_exact(tmp_path):
    src = os.path.join(os.path.dirname(__file__), "csrc", "adj_division_check.c")
    exe = tmp_path / "adjcheck"
    subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-o", str(exe), src, "-lm"])
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout
    assert "bad 0" in out.stdout
