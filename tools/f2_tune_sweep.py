"""Phase times of the one-launch MVM at C2 (32 RHS) under plan tuning keys (GK_TUNE)."""
import os
import subprocess
import sys

here = os.path.dirname(os.path.abspath(__file__))
cfg, nrhs = (sys.argv[1], sys.argv[2]) if len(sys.argv) > 2 else ("C2", "32")
tunes = sys.argv[3].split(";") if len(sys.argv) > 3 else [
    "", "f2_per_sm=4", "f2_sl=10", "f2_sl=7", "f2_nst=4", "f2_stc=16", "f2_nspl=1", "f2_gtc=8", "f2_gl=3",
    "f2_sl=10,f2_stc=4"]
for tune in tunes:
    env = dict(os.environ, GK_TUNE=tune)
    out = subprocess.run([sys.executable, os.path.join(here, "fused_phases.py"), cfg, nrhs], env=env,
                         capture_output=True, text=True)
    lines = [ln for ln in out.stdout.splitlines() if "cumulative" in ln]
    print(f"[{tune}]", *lines, out.stderr[-300:], sep="\n  ", flush=True)
