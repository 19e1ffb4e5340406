for tool in memcheck racecheck synccheck initcheck; do
  echo "== $tool"
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_probe.py 2>&1 | grep -v "^P2\|^C2\|^C1" | tail -8
done
