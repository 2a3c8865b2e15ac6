python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
for e in "8 8 8" "21 21 21" "51 51 51" "50 50 50" "51 51 50"; do timeout 120 python tools/dbg_n4.py 4 $e 2>&1 | grep -E "^ok|Error" | head -2; done
timeout 120 python tools/dbg_n4.py 6 37 37 37 2>&1 | grep -E "^ok|Error" | head -2
timeout 600 compute-sanitizer --tool memcheck python tools/dbg_n4.py 4 21 21 21 2>&1 | grep -v "^=========     Host Frame" | head -40
