"""Print the headline fields of bench JSON lines: python tools/show_bench.py FILE..."""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f"{f.split('/')[-1]:28s} {d['value'] / 1e6:7.1f}M {d['ms_per_step']:7.2f} ms "
              f"pi {d['stage_ms']['pi']:6.2f} nl {d['stage_ms']['nl']:5.3f} su {d['stage_ms']['su']:5.3f} "
              f"lanes {d.get('build', {}).get('pi_lane_use')}")
    except Exception as e:  # noqa: BLE001
        print(f, "ERR", e)
