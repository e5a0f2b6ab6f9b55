"""The scheduled 1-D transforms of csrc/transforms.cuh equal the matrix form (host check)."""
import os
import subprocess
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(os.path.dirname(HERE), "paper_2407_02913_b200", "csrc")


def test_scheduled_transforms_equal_matrix_form():
    with tempfile.TemporaryDirectory() as d:
        exe = os.path.join(d, "check_transforms")
        subprocess.run(["nvcc", "-std=c++17", "-O1", "-x", "cu", f"-I{CSRC}", "-o", exe,
                        os.path.join(HERE, "host", "check_transforms.cu")], check=True)
        r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
