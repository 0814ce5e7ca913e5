"""Print 'a_us,b_ps_per_byte' of a bench JSON line (last line of a log)."""
import json
import sys

c = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])["calibration"]
print(f"{c['a_us']},{c['b_ps_per_byte']}")
