python -m paper_2506_15155_b200.build > /dev/null 2>&1
for rep in 1 2 3; do
for cfg in "split2 0" "split1 1" "split1 0"; do set -- $cfg
  if [ $1 = split1 ]; then export ELLM_LIB_PATH=$PWD/paper_2506_15155_b200/libellm_split1.so; else unset ELLM_LIB_PATH; fi
  echo -n "$1 EMU=$2: "; ELLM_PF_EMU=$2 timeout 300 python tools/prefill_bench.py 2>&1 | tail -5 | awk '{print $(NF-1)}' | tr '\n' ' '; echo
done; done
