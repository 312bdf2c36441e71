"""Print kbench JSON (stdin or file) as one line of name=ms (development tool)."""
import json
import sys

d = json.load(open(sys.argv[1]) if len(sys.argv) > 1 else sys.stdin)
print(" ".join(f"{k}={v['ms']:.4f}" for k, v in d.items() if isinstance(v, dict) and "ms" in v))
