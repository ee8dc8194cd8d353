"""One-line summary of a bench.py JSON line read from stdin (label in argv)."""
import json
import sys

lines = [x for x in sys.stdin.read().strip().splitlines() if x.startswith("{")]
if not lines:
    print(sys.argv[1:], "no JSON line")
    sys.exit(0)
d = json.loads(lines[-1])
r = d.get("roofline_step", {})
rl = d.get("roofline", {})
print(" ".join(sys.argv[1:]), f"{d['value']:.0f} samples/s, {d['ms_per_step']:.2f} ms/step, fwd {r.get('fwd_ms', 0):.2f} "
      f"bwd {r.get('bwd_ms', 0):.2f}, dominant {rl.get('ms', 0):.2f} ms frac {rl.get('frac', 0):.3f}",
      f"e2e {d['e2e']['value']:.0f}" if "e2e" in d else "")
