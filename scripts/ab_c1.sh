#!/bin/bash
# C1 per-elimination time, this tree vs the round-1 tree (scratch_r01/, built
# from commit cfc45be): the same box, back to back.
for tree in . scratch_r01; do
  echo "== tree $tree"
  RPLU_TREE=$tree python scripts/time_c1.py
done
