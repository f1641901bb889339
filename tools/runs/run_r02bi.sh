#!/bin/bash
O=gpurun_out/r02bi
mkdir -p $O
python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
python -c 'import __graft_entry__ as g; g.smoke(); print("smoke ok")' > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
