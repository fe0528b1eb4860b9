"""Sweep onesweep pass variants (NMX_PASS_VARIANT) on device-resident input."""
import os, subprocess, sys
for v in range(8):
    env = dict(os.environ, NMX_PASS_VARIANT=str(v))
    out = subprocess.run([sys.executable, "tools/profile_target.py", sys.argv[1] if len(sys.argv) > 1 else "28"],
                         env=env, capture_output=True, text=True, timeout=300)
    print("variant", v, (out.stdout.strip().splitlines() or ["?"])[-1], out.stderr[-300:], flush=True)
