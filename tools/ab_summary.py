import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "FAILED", open(f).read()[-300:])
        continue
    ks = d["roofline"]["kernels"]
    print(f"{f.split('/')[-1]:28s} {d['ms_per_step']:7.3f} ms  {d['value']/1e9:6.1f} Gunk/s  solve_frac {d['roofline']['solve_frac']:.3f}  "
          f"rel_an {d['parity']['rel_l2_vs_analytic']:.1e}  " + " ".join(f"{k[:5]}={v['ms']:.2f}" for k, v in ks.items()))
