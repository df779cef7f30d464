// b >= 6 team kernels for GenericTraits<8> (fully inlined build; team_launch.cuh).
#include "team_launch.cuh"

using namespace spingp_dev;
using spingp_host::EvalBufs;
using spingp_host::EvalArgs;
SPINGP_TEAM_INST(GenericTraits<8>)
SPINGP_TEAM_UPPER_INST(8)
