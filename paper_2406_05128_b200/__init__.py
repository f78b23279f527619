"""B200-native differentiable time-varying linear prediction (placeholder)."""
