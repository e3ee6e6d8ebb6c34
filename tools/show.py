"""Print the key fields of bench JSON lines in gpurun_out/ (build-box helper)."""
import json, sys
for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(f, "unreadable:", e)
        continue
    keys = ["value", "ms_per_step", "passes", "flagged_rows", "flagged_full_scan_rows", "final_iteration",
            "segments_ms", "rerank_rows_per_step", "roofline", "e2e", "parity", "design", "clocks"]
    print(f, json.dumps({k: d.get(k) for k in keys if d.get(k) is not None})[:1800])
