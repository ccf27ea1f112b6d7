#!/bin/bash
# Steady-state check of the C2 headline: the bench at --steps 10..200 on one box (value must not
# drift with the number of timed rotations; the cache is warmed by 64 untimed rotations first).
mkdir -p gpurun_out
for k in 10 20 50 100 200; do
  timeout 600 python bench.py --steps $k --warmup 5 --no-cpu-baseline --no-standalone \
    > gpurun_out/steps_$k.json 2> gpurun_out/steps_$k.err || echo "steps $k rc=$?"
done
python - <<'PY'
import json
for k in (10, 20, 50, 100, 200):
    try:
        d = json.loads(open(f"gpurun_out/steps_{k}.json").read().strip().splitlines()[-1])
    except Exception as e:
        print(k, "failed", e); continue
    print(json.dumps({"steps": k, "value": round(d["value"]), "e2e": round(d["e2e"]["value"]),
                      "ms_per_step": round(d["ms_per_step"], 2),
                      "cache_hit_token_frac": round(d["cache_hit_token_frac"], 4),
                      "raw_computed_tokens_per_s": round(d["raw_computed_tokens_per_s"]),
                      "sm_mhz": d["clocks"].get("sm_mhz"), "clock_samples": d["clocks"].get("samples"),
                      "reasons": d["clocks"].get("reasons")}))
PY
