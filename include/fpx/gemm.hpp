// include/fpx/gemm.hpp -- reference-layout include path (/root/reference/proj/
// include/fpx/gemm.hpp): a caller written against the reference's headers
// compiles unchanged with -I include and links libfpx_b200.so.  The whole
// drop-in API lives in fpx_b200.hpp.
#pragma once
#include "../fpx_b200.hpp"
