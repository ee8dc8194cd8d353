"""Run pytest node ids one per subprocess with a hard timeout each, streaming
a one-line verdict per node to stdout (GPU-box diagnostics)."""
import subprocess
import sys
import time

timeout = int(sys.argv[1])
for node in sys.argv[2:]:
    t0 = time.time()
    try:
        r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", node], capture_output=True, text=True,
                           timeout=timeout)
        tail = (r.stdout + r.stderr).strip().splitlines()[-12:]
        verdict = "PASS" if r.returncode == 0 else f"FAIL rc={r.returncode}"
    except subprocess.TimeoutExpired as e:
        out = (e.stdout or b"").decode(errors="replace") + (e.stderr or b"").decode(errors="replace")
        tail = out.strip().splitlines()[-12:]
        verdict = "TIMEOUT"
    print(f"== {node}: {verdict} ({time.time() - t0:.1f}s)", flush=True)
    if verdict != "PASS":
        print("\n".join(tail), flush=True)
