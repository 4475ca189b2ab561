# builds and runs the host planning profiler (no GPU needed)
set -e
cd "$(dirname "$0")/../.."
S=paper_2511_21669_b200/csrc
g++ -O2 -std=c++17 -ffp-contract=off ${PROF_FLAGS} -Iinclude -Ithird_party/nlohmann -o /tmp/host_prof tools/scratch/host_prof.cpp \
  $S/host/yaml.cpp $S/host/resolve.cpp $S/host/sweep.cpp $S/host/report.cpp $S/device/pack.cpp $S/host/multi.cpp -lpthread \
  -Wl,--unresolved-symbols=ignore-all
/tmp/host_prof "$@"
