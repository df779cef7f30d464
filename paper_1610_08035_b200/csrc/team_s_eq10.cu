// b >= 6 team kernels for StaticTraits<SEQ<10>> (fully inlined build; team_launch.cuh).
#include "team_launch.cuh"

using namespace spingp_dev;
using spingp_host::EvalBufs;
using spingp_host::EvalArgs;
SPINGP_TEAM_INST(StaticTraits<SEQ<10>>)
SPINGP_TEAM_UPPER_INST(10)
