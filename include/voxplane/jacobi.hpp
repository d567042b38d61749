// Reference-compatible include path (voxplane/jacobi.hpp): the B200 API lives in
// voxplane/voxplane.hpp.
#pragma once
#include "voxplane/voxplane.hpp"
