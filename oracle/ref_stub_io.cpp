// Test infrastructure: stub for the one io symbol the reference hot path links.
// optimize.cpp:452 calls drk::save_scene for periodic checkpoints inside
// train(); scene files are out of scope, so the oracle
// build provides a stub that refuses instead of linking io.cpp (which needs
// the absent nlohmann/json and libpng).
#include <string>

#include "drk/errors.hpp"
#include "drk/io.hpp"

namespace drk {
void save_scene(const Scene&, const std::string& path) {
  throw IoError("save_scene is not part of the oracle build: " + path);
}
}  // namespace drk
