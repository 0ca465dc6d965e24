"""Phase times of the one-launch MVM at C4 / C2 (1 RHS) over Toeplitz m-tile splits."""
import os
import subprocess
import sys

here = os.path.dirname(os.path.abspath(__file__))
for cfg in ("C4", "C2"):
    for ts in (1, 2, 5):
        env = dict(os.environ, GK_TUNE=f"f2_tsplit={ts}")
        out = subprocess.run([sys.executable, os.path.join(here, "fused_phases.py"), cfg, "1"], env=env,
                             capture_output=True, text=True)
        lines = [ln for ln in out.stdout.splitlines() if "cumulative" in ln or "mode" in ln]
        print(f"tsplit={ts}", *lines, out.stderr[-300:], sep="\n  ", flush=True)
