"""Extra GPU fuzz seeds for the JSON / adversarial / Json-kind parity tests (under gpurun)."""
import sys, tempfile
from pathlib import Path
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests"); sys.path.insert(0, "/root/repo/oracle")
import test_gpu_edge as T
ok = 0
for seed in range(int(sys.argv[1]) if len(sys.argv) > 1 else 100, int(sys.argv[2]) if len(sys.argv) > 2 else 112):
    for fn, args in ((T.test_json_fuzz_matches_oracle, (seed,)),
                     (T.test_adversarial_records_match_oracle, (512 if seed % 2 else 100, seed)),
                     (T.test_json_kind_extraction_matches_oracle, (seed,))):
        d = Path(tempfile.mkdtemp())
        try:
            fn(*args, d)
            ok += 1
        except Exception as e:
            print("FAIL", fn.__name__, args, repr(e)[:300])
print("passed", ok)
