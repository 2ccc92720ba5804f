#!/bin/bash
cd tools/abi && timeout 120 ./selftest 2>&1 | tail -20
cd ../..
echo "=== cuda-gdb selftest"
timeout 300 cuda-gdb -batch -ex run -ex bt tools/abi/selftest 2>&1 | tail -30
echo "=== python smoke under gdb"
timeout 300 cuda-gdb -batch -ex run -ex bt --args python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | grep -v "^\[New Thread\|^\[Thread" | tail -40
