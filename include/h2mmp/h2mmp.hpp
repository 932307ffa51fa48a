// Umbrella header of the B200 drop-in for the reference's MMP path.
#pragma once

#include "h2mmp/block_tree.hpp"
#include "h2mmp/cluster_tree.hpp"
#include "h2mmp/dense.hpp"
#include "h2mmp/errors.hpp"
#include "h2mmp/geometry.hpp"
#include "h2mmp/h2_matrix.hpp"
#include "h2mmp/mmp.hpp"
#include "h2mmp/truncation.hpp"
