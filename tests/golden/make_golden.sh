#!/bin/sh
# Regenerates the committed golden fixtures from the reference's own code.
#   rng_kat.json: the reference's proj/include/vlasim/util/rng.hpp compiled as-is
#   (oracle/Makefile target `ref` → oracle/_ref/ref_rng_kat) and run.
set -e
cd "$(dirname "$0")/../.."
make -C oracle ref
./oracle/_ref/ref_rng_kat > tests/golden/rng_kat.json
