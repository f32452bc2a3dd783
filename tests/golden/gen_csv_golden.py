"""Generate tests/golden/csv/*.csv with the REFERENCE's own CSV emitters
(proj/src/csv.cpp) on fixed small inputs: oracle/csv_golden.cpp, built by
`make -C oracle _ref/csv_golden` against the reference's sources where they lie.

    python tests/golden/gen_csv_golden.py

Run in the build container (needs /root/reference); the fixtures travel with
the repo and tests/test_csvio.py compares paper_1510_08982_b200/csvio.py's
output with them byte for byte."""
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
OUT = os.path.join(HERE, "csv")

if __name__ == "__main__":
    subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "_ref/csv_golden"], check=True)
    os.makedirs(OUT, exist_ok=True)
    subprocess.run([os.path.join(ROOT, "oracle", "_ref", "csv_golden"), OUT], check=True)
    print(sorted(os.listdir(OUT)))
