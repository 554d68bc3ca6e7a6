#!/bin/bash
# refresh the serving / trace / verify evidence with the round-2 engine
timeout 300 python tools/serve_sim.py --requests 512 --rate 6 > gpurun_out/r02_serve_sim.json 2> gpurun_out/serve.err
timeout 300 python tools/trace_replay.py --gen c5 --attend --out gpurun_out/r02_trace_replay.jsonl > gpurun_out/trace.log 2>&1
timeout 600 python -m paper_2506_07311_b200.verify > gpurun_out/r02_verify_report.json 2> gpurun_out/verify.err; echo "verify rc=$?"
tail -c 600 gpurun_out/r02_serve_sim.json; echo; tail -3 gpurun_out/trace.log; grep -m3 '"passed"' gpurun_out/r02_verify_report.json
