// Forwarding header: the venv ships only the single-header nlohmann/json 3.11
// (no json_fwd.hpp). Test infrastructure for building oracle/_ref only.
#pragma once
#include <nlohmann/json.hpp>
