#!/bin/bash
# compute-sanitizer over the rewritten codec kernels (toy): memcheck, racecheck, synccheck.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_h.log 2>&1 || { tail -30 gpurun_out/build_h.log; exit 1; }
timeout 300 python scripts/sanitize_codec.py > gpurun_out/san_plain.log 2>&1; echo "plain rc=$?"; tail -1 gpurun_out/san_plain.log
for tool in memcheck racecheck synccheck; do
  echo "== $tool" >> gpurun_out/sanitizer_h.txt
  timeout 1200 compute-sanitizer --tool $tool --kernel-regex kns=inflate,kns=dequant,kns=deflate,kns=section --print-limit 20 python scripts/sanitize_codec.py > gpurun_out/san_$tool.log 2>&1; echo "$tool rc=$?"
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|Error|Race reported|sanitize_codec ok" gpurun_out/san_$tool.log | head -12 >> gpurun_out/sanitizer_h.txt
done
cat gpurun_out/sanitizer_h.txt
