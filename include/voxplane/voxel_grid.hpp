// Reference-compatible include path (voxplane/voxel_grid.hpp): the B200 API lives in
// voxplane/voxplane.hpp.
#pragma once
#include "voxplane/voxplane.hpp"
