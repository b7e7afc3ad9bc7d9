// Tile-local fused V-cycle passes for mid-size levels (mgb_tile.cu).
#pragma once

#include "mgb_stream.h"

namespace mgb {

// Same contract as launch_stream (PRE / plain sweep / POST, nsw in {1, 2}); the
// whole grid is owned (own0 / own1 and seg are ignored).  Bit-identical u and rc.
cudaError_t launch_tile(const StreamArgs& a, int nsw, bool res, bool pro, bool norm, int* nblocks);
int tile_side(const Grid& g);
int tile_max_blocks(const Grid& g);  // upper bound on the CTAs (history partials) per problem

}  // namespace mgb
