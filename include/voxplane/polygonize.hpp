// Reference-compatible include path (voxplane/polygonize.hpp): the B200 API lives in
// voxplane/voxplane.hpp.
#pragma once
#include "voxplane/voxplane.hpp"
