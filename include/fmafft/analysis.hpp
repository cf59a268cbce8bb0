// fmafft/analysis.hpp -- forwarding header of the drop-in: the reference's
// #include "fmafft/analysis.hpp" (proj/core/include/fmafft/analysis.hpp) resolves here
// when this repo's include/ directory precedes the reference's on the include
// path.  Everything lives in include/fmafft_b200.hpp; namespace fmafft names
// it.  Link libdsfft.so (paper_2604_00567_b200/).
#pragma once
#include "../fmafft_b200.hpp"

namespace fmafft = fmafft_b200;
