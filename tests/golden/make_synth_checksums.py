"""Writes tests/golden/synth_checksums.json from synth/ only (never from the CUDA path)."""
import hashlib
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import synth  # noqa: E402

cfg = synth.TINY
out = {"tiny": {s.name: hashlib.sha256(synth.host_shard(cfg, s).tobytes()).hexdigest()
                for s in synth.tensor_specs(cfg)},
       "tiny_prompt0_64": hashlib.sha256(synth.eval_prompt(cfg, 0, 64).tobytes()).hexdigest()}
json.dump(out, open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "synth_checksums.json"), "w"), indent=1)
