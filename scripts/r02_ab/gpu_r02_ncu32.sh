#!/bin/bash
# ncu launch list + one --set full capture per main kernel at the bench's 32-images-per-launch configuration.
set -u
bash scripts/profile_round.sh
