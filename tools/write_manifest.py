"""Write synth/manifest.json: sha256 digests of every BASELINE config's generated inputs
(E, c, queries). Run once when the generator changes on purpose; tests then detect any
unintended change (e.g. a numpy version whose Generator streams differ).

    python tools/write_manifest.py
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

out = {}
for name in synth.CONFIGS:
    wl = synth.make_workload(name)
    out[name] = synth.digest(wl)
    print(name, out[name]["shape"], flush=True)
with open(synth.MANIFEST, "w") as f:
    json.dump(out, f, indent=1, sort_keys=True)
    f.write("\n")
